// C++ drop-in for the reference's batched-RVE entry point on the B200.
//
//   fibra_b200::batch_response(library, assignment, states, law, F, relax_cfg, stiff_cfg, pool)
//
// has the signature and semantics of fibra::batch_response
// (/root/reference/proj/include/fibra/batch.hpp:71-77, src/batch.cpp:155-187): one response per
// point, SolverError/KinematicsError points listed in `failed` (ascending) with
// value-initialized slots, ConfigError thrown, PackedStates mutated in place (warm start in,
// base solution out).  It is header-only over the C-ABI of fibra_cuda.h and compiles inside
// the reference tree (it includes the reference's own headers).  See INTEGRATION.md.
#pragma once

#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "fibra/batch.hpp"
#include "fibra/error.hpp"
#include "fibra_cuda.h"

namespace fibra_b200 {

namespace detail {

// fibra_net_desc views into one reference FiberNetwork plus the arrays the reference keeps
// only as structs (coords, fibers).
struct NetView {
  std::vector<double> coords, area, modulus;
  std::vector<int32_t> fiber_nodes;
  fibra_net_desc desc{};

  explicit NetView(const fibra::FiberNetwork& net) {
    const int n = net.n_nodes(), m = net.n_fibers();
    coords.resize(3 * static_cast<size_t>(n));
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) coords[3 * i + k] = net.coords()[i][k];
    fiber_nodes.resize(2 * static_cast<size_t>(m));
    area.resize(m);
    modulus.resize(m);
    for (int f = 0; f < m; ++f) {
      fiber_nodes[2 * f] = net.fibers()[f].a;
      fiber_nodes[2 * f + 1] = net.fibers()[f].b;
      area[f] = net.fibers()[f].area;
      modulus[f] = net.fibers()[f].modulus;
    }
    desc.n_nodes = n;
    desc.n_fibers = m;
    desc.n_free = net.n_free();
    desc.n_boundary = static_cast<int32_t>(net.boundary_nodes().size());
    desc.coords = coords.data();
    desc.fiber_nodes = fiber_nodes.data();
    desc.fiber_area = area.data();
    desc.fiber_modulus = modulus.data();
    desc.packed_of_dof = net.dof_map().packed_of_dof.data();
    desc.packed_ref = net.packed_ref_coords().data();
    desc.fiber_packed_dofs = net.fiber_packed_dofs().data();
    desc.rest_length = net.rest_lengths().data();
    desc.node_lump = net.node_lumping().data();
    desc.boundary_nodes = net.boundary_nodes().data();
    desc.box_half = net.box().half;
    desc.max_ea = net.max_ea();
  }
};

// One device context per (library, assignment), kept for the thread's lifetime so the
// topology and the warm states stay in HBM between Newton iterations.
struct Ctx {
  fibra_ctx* ctx = nullptr;
  const fibra::RveLibrary* lib = nullptr;
  std::vector<int32_t> eop;
  ~Ctx() { fibra_cuda_close(ctx); }
};

inline void check(int rc, fibra_ctx* ctx) {
  if (rc == FIBRA_OK) return;
  const std::string what = ctx ? fibra_cuda_last_error(ctx) : "fibra_cuda";
  if (rc == FIBRA_E_CONFIG || rc == FIBRA_E_ARG) throw fibra::ConfigError(what);
  if (rc == FIBRA_E_IO) throw fibra::IoError(what);
  throw fibra::Error("B200 solver: " + what);
}

inline Ctx& context(const fibra::RveLibrary& library, const fibra::BatchAssignment& a,
                    int device) {
  thread_local std::map<int, std::unique_ptr<Ctx>> cache;
  auto& slot = cache[device];
  const bool same = slot && slot->lib == &library && slot->eop == a.entry_of_point;
  if (same) return *slot;
  if (!slot || slot->lib != &library) {
    slot = std::make_unique<Ctx>();
    check(fibra_cuda_open(device, &slot->ctx), nullptr);
    std::vector<NetView> views;
    views.reserve(library.entries.size());
    for (const auto& net : library.entries) views.emplace_back(net);
    std::vector<fibra_net_desc> descs;
    for (const auto& v : views) descs.push_back(v.desc);
    check(fibra_cuda_upload_library(slot->ctx, descs.data(), static_cast<int32_t>(descs.size())),
          slot->ctx);
    slot->lib = &library;
  }
  slot->eop = a.entry_of_point;
  check(fibra_cuda_bind_points(slot->ctx, slot->eop.data(), static_cast<int32_t>(slot->eop.size())),
        slot->ctx);
  return *slot;
}

inline fibra::SymTensor3 sym(const double* s) {
  fibra::SymTensor3 t;
  t.xx = s[0];
  t.yy = s[1];
  t.zz = s[2];
  t.yz = s[3];
  t.xz = s[4];
  t.xy = s[5];
  return t;
}

}  // namespace detail

inline fibra::BatchResult batch_response(const fibra::RveLibrary& library,
                                         const fibra::BatchAssignment& assignment,
                                         fibra::PackedStates& states, const fibra::FiberLaw& law,
                                         std::span<const fibra::Def3> deformation,
                                         const fibra::RelaxConfig& relax_cfg,
                                         const fibra::StiffnessConfig& stiff_cfg,
                                         fibra::WorkerPool& /*pool: the GPU grid replaces it*/,
                                         int device = 0) {
  const int n = states.n_points();
  if (static_cast<int>(deformation.size()) != n)
    throw fibra::ConfigError("one deformation gradient per point is required");
  detail::Ctx& c = detail::context(library, assignment, device);
  detail::check(fibra_cuda_upload_states(c.ctx, states.u.data(), states.t.data(),
                                         states.iters.data(), states.converged.data()),
                c.ctx);
  std::vector<double> F(9 * static_cast<size_t>(n));
  for (int p = 0; p < n; ++p)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[9 * p + 3 * i + j] = deformation[p](i, j);
  fibra_law L{law.kind == fibra::FiberLaw::Kind::linear ? 0 : 1, law.ea_scale, law.nonlinearity,
              law.buckling_off ? 1 : 0};
  fibra_relax_cfg R{relax_cfg.damping, relax_cfg.tolerance, relax_cfg.max_iterations,
                    relax_cfg.dt_safety, relax_cfg.density_scale, relax_cfg.energy_check ? 1 : 0};
  fibra_stiff_cfg S{stiff_cfg.fd_rel_step, stiff_cfg.reuse_warm ? 1 : 0};
  std::vector<fibra_point_result> out(n);
  detail::check(fibra_cuda_solve(c.ctx, F.data(), &L, &R, &S, 1, out.data()), c.ctx);
  detail::check(fibra_cuda_download_states(c.ctx, states.u.data(), states.v.data(), states.a.data(),
                                           states.f_int.data(), states.f_damp.data(),
                                           states.mass.data(), states.inv_mass.data(),
                                           states.t.data(), states.iters.data(),
                                           states.converged.data()),
                c.ctx);
  fibra::BatchResult br;
  br.responses.resize(n);
  br.stats.resize(n);
  br.base_reports.resize(n);
  for (int p = 0; p < n; ++p) {
    const fibra_point_result& r = out[p];
    if (r.status != FIBRA_OK) {  // value-initialized slots, id listed (batch.cpp:177-185)
      br.failed.push_back(p);
      continue;
    }
    br.responses[p].sigma = detail::sym(r.sigma);
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) br.responses[p].spatial_c(i, j) = r.spatial_c[6 * i + j];
    br.stats[p].solves = r.solves;
    br.stats[p].relax_iterations = r.relax_iterations;
    br.stats[p].failed_probe = r.failed_probe;
    fibra::RelaxReport& rep = br.base_reports[p];
    rep.iterations = r.base_report.iterations;
    rep.residual = r.base_report.residual;
    rep.eps_eff = r.base_report.eps_eff;
    rep.kinetic_fraction = r.base_report.kinetic_fraction;
    rep.dt = r.base_report.dt;
    rep.converged = r.base_report.converged != 0;
    rep.energy_drift = r.base_report.energy_drift;
  }
  return br;
}

}  // namespace fibra_b200
