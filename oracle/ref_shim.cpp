// ref_shim.cpp -- TEST INFRASTRUCTURE linked with the reference's own, unmodified
// translation units (network.cpp relax.cpp kernels*.cpp netgen.cpp pool.cpp under
// /root/reference/proj/src) into oracle/_ref/libfibra_ref.so.  Nothing here ships.
//
// Two parts:
//  1. The three tensor.cpp symbols those TUs link against, restated because
//     tensor.cpp itself needs Eigen (absent): Def3::det (tensor.cpp:29-33),
//     Def3::apply (:58-62), SymTensor3::from_full (:101-110).
//  2. An extern "C" surface so Python tests and bench.py's reference arm can drive the
//     reference generator, relax_solve, homogenized_stress and WorkerPool directly.
//     The Eigen-dependent polar/pull-back steps of solve_base (stiffness.cpp:66-83) use
//     the oracle restatement (fibra_oracle.c) -- the DR hot loop, force loop, packing
//     and thread pool are the reference's own compiled code.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fibra/error.hpp"
#include "fibra/kernels.hpp"
#include "fibra/netgen.hpp"
#include "fibra/network.hpp"
#include "fibra/pool.hpp"
#include "fibra/relax.hpp"
#include "fibra/tensor.hpp"
#include "fibra_oracle.h"

namespace fibra {

double Def3::det() const {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
         m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

Vec3 Def3::apply(const Vec3& x) const {
  return {m[0][0] * x[0] + m[0][1] * x[1] + m[0][2] * x[2],
          m[1][0] * x[0] + m[1][1] * x[1] + m[1][2] * x[2],
          m[2][0] * x[0] + m[2][1] * x[1] + m[2][2] * x[2]};
}

SymTensor3 SymTensor3::from_full(const Def3& a) {
  SymTensor3 s;
  s.xx = a(0, 0);
  s.yy = a(1, 1);
  s.zz = a(2, 2);
  s.yz = 0.5 * (a(1, 2) + a(2, 1));
  s.xz = 0.5 * (a(0, 2) + a(2, 0));
  s.xy = 0.5 * (a(0, 1) + a(1, 0));
  return s;
}

}  // namespace fibra

namespace {

using namespace fibra;

thread_local std::string g_err;

int classify(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return OR_CONFIG;
  if (dynamic_cast<const KinematicsError*>(&e)) return OR_KINEMATICS;
  if (dynamic_cast<const SolverError*>(&e)) {
    if (g_err.find("collapsed") != std::string::npos) return OR_COLLAPSE;
    if (g_err.find("bad time step") != std::string::npos) return OR_BAD_DT;
    if (g_err.find("diverged") != std::string::npos) return OR_DIVERGED;
    return OR_NOT_CONVERGED;
  }
  return 100;
}

FiberLaw make_law(int kind, double ea_scale, double nonlin, int buckling_off) {
  FiberLaw law;
  law.kind = kind == 0 ? FiberLaw::Kind::linear : FiberLaw::Kind::exponential;
  law.ea_scale = ea_scale;
  law.nonlinearity = nonlin;
  law.buckling_off = buckling_off != 0;
  return law;
}

RelaxConfig make_cfg(const or_relax_cfg* c) {
  RelaxConfig cfg;
  cfg.damping = c->damping;
  cfg.tolerance = c->tolerance;
  cfg.max_iterations = c->max_iterations;
  cfg.dt_safety = c->dt_safety;
  cfg.density_scale = c->density_scale;
  return cfg;
}

Def3 def_of(const double* f) {
  Def3 d;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) d.m[i][j] = f[3 * i + j];
  return d;
}

void copy_report(const RelaxReport& r, or_relax_report* o) {
  o->iterations = r.iterations;
  o->residual = r.residual;
  o->eps_eff = r.eps_eff;
  o->kinetic_fraction = r.kinetic_fraction;
  o->dt = r.dt;
  o->converged = r.converged ? 1 : 0;
  o->energy_drift = r.energy_drift;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate(int style, int nodes, int fibers, double half_length, double merge_radius,
                 int neighbors, double align_bias, const double* align_axis, double area,
                 double modulus, double box_half, double tol_bnd, uint64_t seed,
                 void** out) {
  try {
    NetGenSpec spec;
    spec.style = style == 0 ? NetGenSpec::Style::segments : NetGenSpec::Style::knn;
    spec.nodes = nodes;
    spec.fibers = fibers;
    spec.half_length = half_length;
    spec.merge_radius = merge_radius;
    spec.neighbors = neighbors;
    spec.align_bias = align_bias;
    spec.align_axis = {align_axis[0], align_axis[1], align_axis[2]};
    spec.fiber_area = area;
    spec.fiber_modulus = modulus;
    spec.box.half = box_half;
    spec.tol_bnd = tol_bnd;
    *out = new FiberNetwork(generate_network(spec, seed));
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_network_from_arrays(const double* coords, int n, const int32_t* fa, const int32_t* fb,
                            const double* area, const double* modulus, int m, double box_half,
                            double tol_bnd, void** out) {
  try {
    std::vector<Vec3> c(n);
    for (int i = 0; i < n; ++i) c[i] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
    std::vector<Fiber> f(m);
    for (int i = 0; i < m; ++i) f[i] = {fa[i], fb[i], area[i], modulus[i]};
    RveBox box;
    box.half = box_half;
    *out = new FiberNetwork(std::move(c), std::move(f), box, tol_bnd);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_network_read(const char* path, double box_half, double tol_bnd, void** out) {
  try {
    RveBox box;
    box.half = box_half;
    *out = new FiberNetwork(FiberNetwork::read_file(path, box, tol_bnd));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 10;
  }
}

int ref_network_write(void* h, const char* path) {
  try {
    static_cast<FiberNetwork*>(h)->write_file(path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 10;
  }
}

void ref_network_free(void* h) { delete static_cast<FiberNetwork*>(h); }

void ref_network_sizes(void* h, int* n_nodes, int* n_fibers, int* n_free, int* n_boundary) {
  const FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  *n_nodes = net.n_nodes();
  *n_fibers = net.n_fibers();
  *n_free = net.n_free();
  *n_boundary = static_cast<int>(net.boundary_nodes().size());
}

void ref_network_export(void* h, double* coords, int32_t* fa, int32_t* fb, double* area,
                        double* modulus, double* rest_length, int32_t* boundary_nodes,
                        int32_t* packed_of_dof, double* packed_ref, int32_t* fiber_dofs,
                        double* node_lump, double* max_ea) {
  const FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  for (int i = 0; i < net.n_nodes(); ++i)
    for (int k = 0; k < 3; ++k) coords[3 * i + k] = net.coords()[i][k];
  for (int f = 0; f < net.n_fibers(); ++f) {
    fa[f] = net.fibers()[f].a;
    fb[f] = net.fibers()[f].b;
    area[f] = net.fibers()[f].area;
    modulus[f] = net.fibers()[f].modulus;
    rest_length[f] = net.rest_length(f);
  }
  std::memcpy(boundary_nodes, net.boundary_nodes().data(),
              sizeof(int32_t) * net.boundary_nodes().size());
  std::memcpy(packed_of_dof, net.dof_map().packed_of_dof.data(), sizeof(int32_t) * net.n_dof());
  std::memcpy(packed_ref, net.packed_ref_coords().data(), sizeof(double) * net.n_dof());
  std::memcpy(fiber_dofs, net.fiber_packed_dofs().data(), sizeof(int32_t) * 6 * net.n_fibers());
  std::memcpy(node_lump, net.node_lumping().data(), sizeof(double) * net.n_nodes());
  *max_ea = net.max_ea();
}

int ref_relax_solve(void* h, int law_kind, double ea_scale, double nonlin, int buckling_off,
                    const double* F, const or_relax_cfg* cfg, double* u, double* v, double* a,
                    double* f_int, double* f_damp, double* mass, double* inv_mass, double* t,
                    int64_t* iters, uint8_t* converged, int warm_reuse, or_relax_report* rep) {
  const FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  const std::size_t nd = static_cast<std::size_t>(net.n_dof());
  RveStateView s;
  s.u = std::span<double>(u, nd);
  s.v = std::span<double>(v, nd);
  s.a = std::span<double>(a, nd);
  s.f_int = std::span<double>(f_int, nd);
  s.f_damp = std::span<double>(f_damp, nd);
  s.mass = std::span<double>(mass, nd);
  s.inv_mass = std::span<double>(inv_mass, nd);
  s.t = t;
  s.iters = iters;
  s.converged = converged;
  s.n_free = net.n_free();
  try {
    const RelaxReport r = relax_solve(net, make_law(law_kind, ea_scale, nonlin, buckling_off),
                                      def_of(F), make_cfg(cfg), s,
                                      warm_reuse ? WarmStart::reuse : WarmStart::zero_interior);
    copy_report(r, rep);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// the reference's own orientation_p2 (network.cpp:398-415)
double ref_orientation_p2(void* h, const double* u, const double* dir) {
  FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  const std::span<const double> uu(u, static_cast<std::size_t>(net.n_dof()));
  return orientation_p2(net, uu, Vec3{dir[0], dir[1], dir[2]});
}

int ref_homogenized_stress(void* h, const double* u, const double* f_int, int converged,
                           const double* F, double* sigma6, double* asym) {
  FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  const std::size_t nd = static_cast<std::size_t>(net.n_dof());
  std::vector<double> uu(u, u + nd), ff(f_int, f_int + nd);
  uint8_t conv = static_cast<uint8_t>(converged);
  RveStateView s;
  s.u = uu;
  s.f_int = ff;
  s.converged = &conv;
  s.n_free = net.n_free();
  try {
    const HomogenizedStress hs = homogenized_stress(net, s, def_of(F), net.box());
    const double out[6] = {hs.sigma.xx, hs.sigma.yy, hs.sigma.zz,
                           hs.sigma.yz, hs.sigma.xz, hs.sigma.xy};
    std::memcpy(sigma6, out, sizeof out);
    *asym = hs.asymmetry;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_internal_forces(void* h, int law_kind, double ea_scale, double nonlin,
                        int buckling_off, const double* u, double* f_int) {
  const FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  const std::size_t nd = static_cast<std::size_t>(net.n_dof());
  try {
    internal_forces(net, make_law(law_kind, ea_scale, nonlin, buckling_off),
                    std::span<const double>(u, nd), std::span<double>(f_int, nd));
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_select_isa(int avx2) {
  try {
    kernels::select(avx2 ? kernels::Isa::avx2 : kernels::Isa::scalar);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_active_isa() { return kernels::active_isa() == kernels::Isa::avx2 ? 1 : 0; }

// Stress-only batch (the base half of constitutive_response, stiffness.cpp:153-175)
// dispatched one point per task through the reference WorkerPool (pool.cpp:75-99),
// exactly like batch_response (batch.cpp:169-182).  Fresh states per call
// (init_batch zero-fills, batch.cpp:134-143).  Outputs: sigma (n x 6, rotated into the
// frame of F), base iterations and a status per point.
int ref_batch_stress(void* h, int n_points, const double* F, int law_kind, double ea_scale,
                     double nonlin, int buckling_off, const or_relax_cfg* cfg, int workers,
                     double* sigma_out, int64_t* iters_out, int32_t* status) {
  const FiberNetwork& net = *static_cast<FiberNetwork*>(h);
  const FiberLaw law = make_law(law_kind, ea_scale, nonlin, buckling_off);
  const RelaxConfig rc = make_cfg(cfg);
  const std::size_t nd = static_cast<std::size_t>(net.n_dof());
  try {
    WorkerPool pool(workers);
    pool.run(n_points, [&](int p) {
      std::vector<double> buf(7 * nd, 0.0);
      double t = 0;
      std::int64_t it = 0;
      std::uint8_t conv = 0;
      RveStateView s;
      s.u = std::span<double>(buf.data(), nd);
      s.v = std::span<double>(buf.data() + nd, nd);
      s.a = std::span<double>(buf.data() + 2 * nd, nd);
      s.f_int = std::span<double>(buf.data() + 3 * nd, nd);
      s.f_damp = std::span<double>(buf.data() + 4 * nd, nd);
      s.mass = std::span<double>(buf.data() + 5 * nd, nd);
      s.inv_mass = std::span<double>(buf.data() + 6 * nd, nd);
      s.t = &t;
      s.iters = &it;
      s.converged = &conv;
      s.n_free = net.n_free();
      double R[9], U[6], fu9[9];
      status[p] = 0;
      iters_out[p] = 0;
      std::memset(sigma_out + 6 * p, 0, 6 * sizeof(double));
      int rc2 = or_polar_decompose(F + 9 * p, R, U);
      if (rc2) { status[p] = rc2; return; }
      or_sym_full(U, fu9);
      try {
        const RelaxReport r = relax_solve(net, law, def_of(fu9), rc, s, WarmStart::reuse);
        iters_out[p] = r.iterations;
        if (!r.converged) { status[p] = OR_NOT_CONVERGED; return; }
        const HomogenizedStress hs = homogenized_stress(net, s, def_of(fu9), net.box());
        const double su6[6] = {hs.sigma.xx, hs.sigma.yy, hs.sigma.zz,
                               hs.sigma.yz, hs.sigma.xz, hs.sigma.xy};
        double su[9], rt[9], t1[9], s9[9];
        or_sym_full(su6, su);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) rt[3 * i + j] = R[3 * j + i];
        or_matmul(R, su, t1);
        or_matmul(t1, rt, s9);
        or_sym_from_full(s9, sigma_out + 6 * p);
      } catch (const SolverError& e) {
        status[p] = classify(e);
      } catch (const KinematicsError& e) {
        status[p] = classify(e);
      }
    });
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}


// Full constitutive_response (stiffness.cpp:153-175: solve_base :66-83, probe_pk2s :86-123,
// material_stiffness_from_probes :15-41, push_forward_stiffness tensor.cpp:286-300) per
// point through the reference WorkerPool: every one of the 7 DR solves and every
// homogenized stress is the reference's compiled relax_solve / homogenized_stress; the
// Eigen/tensor.cpp steps (polar, pull-back, probing, FullPivLU, push-forward) come from the
// oracle restatement.  Fresh states (init_batch).  Per point: sigma[6], spatial C[36],
// base iterations, relax_iterations (all solves), solves, failed_probe, status.
int ref_batch_response(void* const* nets, const int32_t* entry_of_point, int n_points,
                       const double* F, int law_kind, double ea_scale, double nonlin,
                       int buckling_off, const or_relax_cfg* cfg, double fd_rel_step,
                       int reuse_warm, int want_tangent, int workers, double* sigma_out,
                       double* c_out, int64_t* base_iters, int64_t* relax_iters,
                       int32_t* solves, int32_t* failed_probe, int32_t* status) {
  const FiberLaw law = make_law(law_kind, ea_scale, nonlin, buckling_off);
  const RelaxConfig rc = make_cfg(cfg);
  struct Buf {
    std::vector<double> b;
    double t = 0;
    std::int64_t it = 0;
    std::uint8_t conv = 0;
    RveStateView view(std::size_t nd, int n_free) {
      b.assign(7 * nd, 0.0);
      RveStateView s;
      s.u = std::span<double>(b.data(), nd);
      s.v = std::span<double>(b.data() + nd, nd);
      s.a = std::span<double>(b.data() + 2 * nd, nd);
      s.f_int = std::span<double>(b.data() + 3 * nd, nd);
      s.f_damp = std::span<double>(b.data() + 4 * nd, nd);
      s.mass = std::span<double>(b.data() + 5 * nd, nd);
      s.inv_mass = std::span<double>(b.data() + 6 * nd, nd);
      s.t = &t;
      s.iters = &it;
      s.converged = &conv;
      s.n_free = n_free;
      return s;
    }
  };
  try {
    WorkerPool pool(workers);
    pool.run(n_points, [&](int p) {
      const FiberNetwork& net = *static_cast<const FiberNetwork*>(nets[entry_of_point[p]]);
      const std::size_t nd = static_cast<std::size_t>(net.n_dof());
      double* sig = sigma_out + 6 * p;
      double* cc = c_out + 36 * p;
      std::memset(sig, 0, 6 * sizeof(double));
      std::memset(cc, 0, 36 * sizeof(double));
      base_iters[p] = relax_iters[p] = 0;
      solves[p] = 0;
      failed_probe[p] = -1;
      status[p] = 0;
      Buf base, scratch;
      RveStateView s = base.view(nd, net.n_free());
      double R[9], U[6], fu9[9], su6[6], pk2[6];
      int rc2 = or_polar_decompose(F + 9 * p, R, U);
      if (rc2) { status[p] = rc2; return; }
      or_sym_full(U, fu9);
      try {
        const RelaxReport r = relax_solve(net, law, def_of(fu9), rc, s, WarmStart::reuse);
        base_iters[p] = r.iterations;
        if (!r.converged) { status[p] = OR_NOT_CONVERGED; return; }
        const HomogenizedStress hs = homogenized_stress(net, s, def_of(fu9), net.box());
        const double a6[6] = {hs.sigma.xx, hs.sigma.yy, hs.sigma.zz,
                              hs.sigma.yz, hs.sigma.xz, hs.sigma.xy};
        std::memcpy(su6, a6, sizeof a6);
        if ((rc2 = or_pull_back_stress(su6, fu9, pk2))) { status[p] = rc2; return; }
        solves[p] = 1;
        relax_iters[p] = r.iterations;
      } catch (const SolverError& e) {
        status[p] = classify(e);
        return;
      } catch (const KinematicsError& e) {
        status[p] = classify(e);
        return;
      }
      if (want_tangent) {
        const double h = fd_rel_step * std::sqrt(U[0] * U[0] + U[1] * U[1] + U[2] * U[2] +
                                                 2.0 * (U[3] * U[3] + U[4] * U[4] + U[5] * U[5]));
        RveStateView sc = scratch.view(nd, net.n_free());
        double probes[36];
        for (int q = 0; q < 6; ++q) {
          double dir[6], up[6], fq[9];
          or_probing_direction(q, dir);
          for (int i = 0; i < 6; ++i) up[i] = U[i] + dir[i] * h;
          or_sym_full(up, fq);
          if (!(or_det(fq) > 0)) { status[p] = OR_PROBE_FAILED; return; }
          if (reuse_warm) std::copy(s.u.begin(), s.u.end(), sc.u.begin());
          try {
            const RelaxReport pr = relax_solve(net, law, def_of(fq), rc, sc,
                                               reuse_warm ? WarmStart::reuse : WarmStart::zero_interior);
            ++solves[p];
            relax_iters[p] += pr.iterations;
            if (!pr.converged) { failed_probe[p] = q; status[p] = OR_PROBE_FAILED; return; }
            const HomogenizedStress hq = homogenized_stress(net, sc, def_of(fq), net.box());
            const double q6[6] = {hq.sigma.xx, hq.sigma.yy, hq.sigma.zz,
                                  hq.sigma.yz, hq.sigma.xz, hq.sigma.xy};
            if ((rc2 = or_pull_back_stress(q6, fq, probes + 6 * q))) { status[p] = rc2; return; }
          } catch (const SolverError& e) {
            failed_probe[p] = q;
            status[p] = OR_PROBE_FAILED;
            return;
          }
        }
        double a[36];
        if ((rc2 = or_material_stiffness_from_probes(U, pk2, probes, h, a))) { status[p] = rc2; return; }
        if ((rc2 = or_push_forward_stiffness(a, F + 9 * p, cc))) { status[p] = rc2; return; }
      }
      double su[9], rt[9], t1[9], s9[9];
      or_sym_full(su6, su);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rt[3 * i + j] = R[3 * j + i];
      or_matmul(R, su, t1);
      or_matmul(t1, rt, s9);
      or_sym_from_full(s9, sig);
    });
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

}  // extern "C"
