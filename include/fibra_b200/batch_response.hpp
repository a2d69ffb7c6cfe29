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

#include <cstdint>
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

// FNV-1a over the words of every array the upload reads: the context cache is keyed on the
// library's CONTENT (a library edited in place, or a new one at a recycled address, is
// re-uploaded), not on its address.
inline uint64_t mix(uint64_t h, const void* p, size_t bytes) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  size_t i = 0;
  for (; i + 8 <= bytes; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 0x100000001b3ull;
  }
  for (; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

template <class V>
uint64_t mix_vec(uint64_t h, const V& v) {
  const uint64_t n = v.size();
  h = mix(h, &n, sizeof n);
  return v.empty() ? h : mix(h, v.data(), v.size() * sizeof(v[0]));
}

inline uint64_t library_key(const fibra::RveLibrary& library) {
  uint64_t h = 0xcbf29ce484222325ull;
  const uint64_t n = library.entries.size();
  h = mix(h, &n, sizeof n);
  for (const fibra::FiberNetwork& net : library.entries) {
    const int32_t sz[3] = {net.n_nodes(), net.n_fibers(), net.n_free()};
    h = mix(h, sz, sizeof sz);
    h = mix_vec(h, net.coords());
    for (const fibra::Fiber& f : net.fibers()) {
      h = mix(h, &f.a, sizeof f.a);
      h = mix(h, &f.b, sizeof f.b);
      h = mix(h, &f.area, sizeof f.area);
      h = mix(h, &f.modulus, sizeof f.modulus);
    }
    h = mix_vec(h, net.packed_ref_coords());
    h = mix_vec(h, net.rest_lengths());
    h = mix_vec(h, net.node_lumping());
    const double box = net.box().half;
    h = mix(h, &box, sizeof box);
  }
  return h;
}

// One device context per (library content, assignment), kept for the thread's lifetime so
// the topology and the warm states stay in HBM between Newton iterations.
struct Ctx {
  fibra_ctx* ctx = nullptr;
  uint64_t key = 0;
  std::vector<int32_t> eop;
  std::vector<int64_t> offsets;  // PackedStates layout of the bound points
  ~Ctx() { fibra_cuda_close(ctx); }
};

inline void check(int rc, fibra_ctx* ctx) {
  if (rc == FIBRA_OK) return;
  const std::string what = ctx ? fibra_cuda_last_error(ctx) : "fibra_cuda";
  if (rc == FIBRA_E_CONFIG || rc == FIBRA_E_ARG) throw fibra::ConfigError(what);
  if (rc == FIBRA_E_IO) throw fibra::IoError(what);
  throw fibra::Error("B200 solver: " + what);
}

inline void upload(Ctx& c, const fibra::RveLibrary& library) {
  std::vector<NetView> views;
  views.reserve(library.entries.size());
  for (const auto& net : library.entries) views.emplace_back(net);
  std::vector<fibra_net_desc> descs;
  for (const auto& v : views) descs.push_back(v.desc);
  check(fibra_cuda_upload_library(c.ctx, descs.data(), static_cast<int32_t>(descs.size())),
        c.ctx);
}

inline void bind(Ctx& c, const fibra::RveLibrary& library, const fibra::BatchAssignment& a) {
  const int n = static_cast<int>(a.entry_of_point.size());
  for (int32_t e : a.entry_of_point)
    if (e < 0 || e >= static_cast<int>(library.entries.size()))
      throw fibra::ConfigError("assignment names an entry outside the RVE library");
  c.eop = a.entry_of_point;
  c.offsets.assign(n + 1, 0);
  for (int p = 0; p < n; ++p)
    c.offsets[p + 1] = c.offsets[p] + library.entries[c.eop[p]].n_dof();
  check(fibra_cuda_bind_points(c.ctx, c.eop.data(), n), c.ctx);
}

// The PackedStates must have the layout init_batch gives this library and assignment
// (batch.cpp:94-145); relax_solve throws ConfigError("state layout does not match the
// network") otherwise (relax.cpp:99-100), and so do we -- before any host buffer is read.
inline void check_layout(const Ctx& c, const fibra::PackedStates& st) {
  const size_t n = c.eop.size();
  const int64_t tot = c.offsets.back();
  const auto dofs = [&](const std::vector<double>& v) { return static_cast<int64_t>(v.size()) == tot; };
  if (st.offsets != c.offsets || !dofs(st.u) || !dofs(st.v) || !dofs(st.a) || !dofs(st.f_int) ||
      !dofs(st.f_damp) || !dofs(st.mass) || !dofs(st.inv_mass) || st.t.size() != n ||
      st.iters.size() != n || st.converged.size() != n)
    throw fibra::ConfigError("state layout does not match the network");
}

// open one device, or several GPUs of this process (fibra_cuda_open_devices)
inline int open_ctx(const std::vector<int32_t>& devices, fibra_ctx** out) {
  if (devices.size() == 1) return fibra_cuda_open(devices[0], out);
  return fibra_cuda_open_devices(devices.data(), static_cast<int32_t>(devices.size()), out);
}

inline Ctx& context(const fibra::RveLibrary& library, const fibra::BatchAssignment& a,
                    const std::vector<int32_t>& devices) {
  thread_local std::map<std::vector<int32_t>, std::unique_ptr<Ctx>> cache;
  auto& slot = cache[devices];
  const uint64_t key = library_key(library);
  if (!slot || slot->key != key) {
    slot = std::make_unique<Ctx>();
    check(open_ctx(devices, &slot->ctx), nullptr);
    upload(*slot, library);
    slot->key = key;
    slot->eop.clear();
  }
  if (slot->eop.empty() || slot->eop != a.entry_of_point) bind(*slot, library, a);
  return *slot;
}

inline void to_cfg(const fibra::FiberLaw& law, const fibra::RelaxConfig& relax_cfg,
                   const fibra::StiffnessConfig& stiff_cfg, fibra_law& L, fibra_relax_cfg& R,
                   fibra_stiff_cfg& S) {
  L = fibra_law{law.kind == fibra::FiberLaw::Kind::linear ? 0 : 1, law.ea_scale,
                law.nonlinearity, law.buckling_off ? 1 : 0};
  R = fibra_relax_cfg{relax_cfg.damping, relax_cfg.tolerance, relax_cfg.max_iterations,
                      relax_cfg.dt_safety, relax_cfg.density_scale,
                      relax_cfg.energy_check ? 1 : 0};
  S = fibra_stiff_cfg{stiff_cfg.fd_rel_step, stiff_cfg.reuse_warm ? 1 : 0};
}

inline std::vector<double> flat_F(std::span<const fibra::Def3> deformation) {
  std::vector<double> F(9 * deformation.size());
  for (size_t p = 0; p < deformation.size(); ++p)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[9 * p + 3 * i + j] = deformation[p](i, j);
  return F;
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


// Records -> BatchResult (batch.cpp:169-186): failed points keep value-initialized slots.
inline fibra::BatchResult to_result(const std::vector<fibra_point_result>& out) {
  const int n = static_cast<int>(out.size());
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
    br.responses[p].sigma = sym(r.sigma);
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

}  // namespace detail

inline fibra::BatchResult batch_response(const fibra::RveLibrary& library,
                                         const fibra::BatchAssignment& assignment,
                                         fibra::PackedStates& states, const fibra::FiberLaw& law,
                                         std::span<const fibra::Def3> deformation,
                                         const fibra::RelaxConfig& relax_cfg,
                                         const fibra::StiffnessConfig& stiff_cfg,
                                         fibra::WorkerPool& /*pool: the GPU grid replaces it*/,
                                         const std::vector<int32_t>& devices) {
  const int n = states.n_points();
  if (devices.empty()) throw fibra::ConfigError("no device");
  if (static_cast<int>(deformation.size()) != n)
    throw fibra::ConfigError("one deformation gradient per point is required");
  if (static_cast<int>(assignment.entry_of_point.size()) != n)
    throw fibra::ConfigError("assignment does not match the packed states");
  detail::Ctx& c = detail::context(library, assignment, devices);
  detail::check_layout(c, states);
  detail::check(fibra_cuda_upload_states(c.ctx, states.u.data(), states.t.data(),
                                         states.iters.data(), states.converged.data()),
                c.ctx);
  const std::vector<double> F = detail::flat_F(deformation);
  fibra_law L;
  fibra_relax_cfg R;
  fibra_stiff_cfg S;
  detail::to_cfg(law, relax_cfg, stiff_cfg, L, R, S);
  std::vector<fibra_point_result> out(n);
  detail::check(fibra_cuda_solve(c.ctx, F.data(), &L, &R, &S, 1, out.data()), c.ctx);
  detail::check(fibra_cuda_download_states(c.ctx, states.u.data(), states.v.data(), states.a.data(),
                                           states.f_int.data(), states.f_damp.data(),
                                           states.mass.data(), states.inv_mass.data(),
                                           states.t.data(), states.iters.data(),
                                           states.converged.data()),
                c.ctx);
  return detail::to_result(out);
}

// one B200 (device index) -- the reference signature plus an optional device
inline fibra::BatchResult batch_response(const fibra::RveLibrary& library,
                                         const fibra::BatchAssignment& assignment,
                                         fibra::PackedStates& states, const fibra::FiberLaw& law,
                                         std::span<const fibra::Def3> deformation,
                                         const fibra::RelaxConfig& relax_cfg,
                                         const fibra::StiffnessConfig& stiff_cfg,
                                         fibra::WorkerPool& pool, int device = 0) {
  return batch_response(library, assignment, states, law, deformation, relax_cfg, stiff_cfg,
                        pool, std::vector<int32_t>{device});
}

}  // namespace fibra_b200
