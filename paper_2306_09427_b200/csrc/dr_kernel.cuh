// Persistent dynamic-relaxation kernel: one CTA solves one RVE at a time, pulling
// (point, solve) tickets from a device queue until the batch is drained.
//
// Reference path this replaces (paths under /root/reference/proj):
//   relax_solve           src/relax.cpp:93-191   (setup :95-145, hot loop :148-179)
//   internal_forces_cfl   src/network.cpp:275-324 (force law :16-53)
//   L1 kernels            src/kernels_scalar.cpp:7-65 (contract include/fibra/kernels.hpp:8-15)
//   apply_affine_bc       src/network.cpp:254-269
//   homogenized_stress    src/network.cpp:341-372
//   probe_pk2s            src/stiffness.cpp:86-123 (probes are tickets n..7n-1)
//
// Bitwise contract with the reference: compiled with --fmad=false,
// IEEE div/sqrt; x = ref + u rounded per node; each node's force is accumulated from +0.0
// over its incident fibers in ascending fiber id (CSR, no atomics), reproducing
// f[a] -= g*d / f[b] += g*d of network.cpp:298-303; the damped update follows
// kernels_scalar.cpp:15-17 and relax.cpp:155-166 literally.
//
// Per DR iteration the CTA runs two phases separated by __syncthreads():
//   fiber phase: each thread evaluates FPT register-resident fibers from x in shared
//                memory and writes g*d (SoA) to shared memory;
//   node phase:  each thread owns NPT nodes (state u, v, a, f, f_damp in registers),
//                gathers its CSR list, applies the damped central-difference update and
//                writes the next x.
// The convergence reduction of iteration k is off the critical path: node threads store
// one |f|^2 partial per node, and during fiber phase k+1 the last warp reduces them
// (tree order) and publishes the decision; node phase k+1 acts on it and, if iteration k
// converged, emits the state of iteration k (held in registers), discarding the
// speculative step.  A tree sum differs from the reference's 4-lane interleaved sum
// (kernels_scalar.cpp:20-33) in the last ulps, so whenever |R - eps| <= 1e-10 eps (or a
// value is non-finite) the CTA recomputes both norms in the reference order before
// deciding; the reported residual/eps_eff are always the reference-order values.
#pragma once

#include <cstdint>

#include "fibra_cuda.h"
#include "tensor.cuh"

namespace fibra_b200 {

struct EntryDev {        // one RveLibrary entry in HBM (batched SoA + CSR)
  int n_nodes, n_fibers, n_free_nodes, pad0;
  double max_lump, max_ea, box_volume, pad1;
  const double* ref;     // 3N, packed DOF order (node pn owns dofs 3pn..3pn+2)
  const double* lump;    // N, packed node order
  const int* fiber_ab;   // M, a | b << 16 (packed node ids)
  const double* l0;      // M rest lengths
  const double* ea;      // M area*modulus
  const int* csr_off;    // N+1
  const int* csr_ent;    // 2M, fiber << 1 | (node is endpoint a)
};

struct SolveOut {        // one DR solve (base or probe)
  double sigma_u[6];
  double asym;
  double pk2[6];
  long long iterations;
  double residual, eps_eff, kinetic_fraction, dt;
  int converged;
  int status;
};

struct DrParams {
  const EntryDev* entries;
  const int* entry_of_point;
  const long long* offsets;
  double *u, *v, *a, *f_int, *f_damp, *mass, *inv_mass, *t;
  long long* iters;
  unsigned char* converged;
  const double* solve_F;       // 9 per solve
  const int* solve_skip;       // nonzero: solve pre-failed by prep (status code)
  SolveOut* out;
  int* base_flag;              // per point: 0 pending, 1 converged, 2 failed
  int* ticket;
  unsigned long long* counters;  // [0] iterations [1] fiber-iterations [2] pipe ops [3] solves
  int n_points, n_solves;
  int nmax, mmax;              // smem layout capacity
  int reuse_warm;
  int law_buckling_off;
  double ea_scale, nonlinearity;
  double damping, tolerance, dt_safety, density_scale;
  long long max_iterations;
};

enum : int { kDecConv = 1, kDecExact = 2, kDecNonfinite = 4 };

struct __align__(16) DrCtl {
  int solve, point, q, entry;
  int flag, collapse, pad0, pad1;
  int dec;
  double dec_res, dec_eps;
  double warp_min[32];
  double ex[12];
  double t;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = smin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double flip(double x, int neg) {  // x or -x, exact
  return __longlong_as_double(__double_as_longlong(x) ^ (static_cast<long long>(neg) << 63));
}

// axial force N(lambda) and tangent (network.cpp:16-38); s = ea_scale*ea
template <int LAW>
__device__ __forceinline__ double law_force(double s, double stretch, int buckling_off,
                                            double B) {
  if (buckling_off && stretch < 1.0) return 0.0;
  if (LAW == 0) return s * (stretch - 1.0);
  return s / B * expm1(B * (stretch - 1.0));
}

template <int LAW>
__device__ __forceinline__ double law_tangent(double s, double stretch, int buckling_off,
                                              double B) {
  if (buckling_off && stretch < 1.0) return 0.0;
  if (LAW == 0) return s;
  return s * exp(B * (stretch - 1.0));
}

template <int LAW>
__device__ __forceinline__ double law_energy(double s, double stretch, double rl,
                                             int buckling_off, double B) {  // :40-53
  if (buckling_off && stretch < 1.0) return 0.0;
  const double e = stretch - 1.0;
  if (LAW == 0) return 0.5 * s * rl * e * e;
  return rl * s / B * (expm1(B * e) / B - e);
}

template <int T, int FPT, int NPT, int LAW>
__global__ void __launch_bounds__(T, (T <= 256 ? 2 : 1)) dr_persistent_kernel(DrParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ DrCtl ctl;
  constexpr int NW = T / 32;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // shared layout: [A: 3*nmax x SoA / exact scratch][B: gd SoA 3*mmax | exit scratch]
  //                [spart: nmax][csr_off: nmax+1][csr_ent: 2*mmax]
  const int nmax = P.nmax, mmax = P.mmax;
  const int bsize = (3 * mmax > 6 * nmax + mmax) ? 3 * mmax : 6 * nmax + mmax;
  double* sx = reinterpret_cast<double*>(smem_raw);
  double* sy = sx + nmax;
  double* sz = sy + nmax;
  double* regB = sz + nmax;
  double* gx = regB;
  double* gy = gx + mmax;
  double* gz = gy + mmax;
  double* spart = regB + bsize;
  int* coff = reinterpret_cast<int*>(spart + nmax);
  int* cent = coff + nmax + 1;

  const double B = P.nonlinearity;
  const int bo = P.law_buckling_off;

  // register-resident topology of the loaded entry
  int fab[FPT];
  double fl0[FPT], fs[FPT], fthr[FPT], fmred[FPT];
  int nbeg[NPT], nend[NPT];
  double nref[NPT][3], nm[NPT], ninv[NPT], ncm[NPT];
  int cur_entry = -1;
  int N = 0, M = 0, NFN = 0;
  double max_lump = 1, force_floor = 0, box_volume = 1;

  for (;;) {
    if (tid == 0) {
      const int s = atomicAdd(P.ticket, 1);
      ctl.solve = s;
      if (s < P.n_solves) {
        const int p = s < P.n_points ? s : (s - P.n_points) / 6;
        ctl.point = p;
        ctl.q = s < P.n_points ? -1 : (s - P.n_points) % 6;
        ctl.entry = P.entry_of_point[p];
        ctl.collapse = 0;
        int flag = 1;
        if (P.solve_skip[s]) {
          flag = 0;
        } else if (ctl.q >= 0) {  // probe: wait for the base solve of its point
          int f;
          while ((f = ld_acquire(P.base_flag + p)) == 0) __nanosleep(256);
          flag = (f == 1);
        }
        ctl.flag = flag;
      }
    }
    __syncthreads();
    const int s = ctl.solve;
    if (s >= P.n_solves) break;
    const int p = ctl.point, q = ctl.q, e = ctl.entry;
    if (!ctl.flag) {  // pre-failed (prep) or base failed: nothing to solve
      if (tid == 0) {
        SolveOut o = {};
        o.status = P.solve_skip[s] ? P.solve_skip[s] : FIBRA_E_NOT_CONVERGED;
        P.out[s] = o;
        if (q < 0) {
          __threadfence();
          atomicExch(P.base_flag + p, 2);
        }
      }
      __syncthreads();
      continue;
    }

    const EntryDev& E = P.entries[e];
    const double scale = P.density_scale / E.max_lump;  // setup_mass relax.cpp:35-43
    if (e != cur_entry) {
      cur_entry = e;
      N = E.n_nodes;
      M = E.n_fibers;
      NFN = E.n_free_nodes;
      max_lump = E.max_lump;
      box_volume = E.box_volume;
      force_floor = P.ea_scale * E.max_ea * 1e-12;  // relax.cpp:112
      for (int i = tid; i <= N; i += T) coff[i] = E.csr_off[i];
      for (int i = tid; i < 2 * M; i += T) cent[i] = E.csr_ent[i];
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = j * T + tid;
        if (f < M) {
          fab[j] = E.fiber_ab[f];
          fl0[j] = E.l0[f];
          fs[j] = P.ea_scale * E.ea[f];
          fthr[j] = 1e-8 * fl0[j];
        }
      }
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int pn = j * T + tid;
        if (pn < N) {
          nbeg[j] = E.csr_off[pn];
          nend[j] = E.csr_off[pn + 1];
          nref[j][0] = E.ref[3 * pn];
          nref[j][1] = E.ref[3 * pn + 1];
          nref[j][2] = E.ref[3 * pn + 2];
        }
      }
    }
    (void)max_lump;
    // ---- per-solve setup (relax.cpp:95-145) ----
    const double* F = P.solve_F + 9 * s;
    double Fm[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fm[i] = F[i];
    const long long off = P.offsets[p];
    const bool is_base = q < 0;
    double lmin = INFINITY;
#pragma unroll
    for (int j = 0; j < FPT; ++j) {
      const int f = j * T + tid;
      if (f < M) {  // reduced_mass_l0 relax.cpp:46-55; CFL at stretch-independent kt
        const double ma = E.lump[fab[j] & 0xffff] * scale;
        const double mb = E.lump[fab[j] >> 16] * scale;
        fmred[j] = ma * mb / (ma + mb) * fl0[j];
        if (LAW == 0) {
          const double kt = smax(fabs(law_tangent<0>(fs[j], 1.0, 0, B)), fs[j]);
          lmin = smin(lmin, fmred[j] / kt);
        }
      }
    }
    double u[NPT][3], vh[NPT][3];                       // current (speculative) state
    double pu[NPT][3], pv[NPT][3], pa[NPT][3], pf[NPT][3], pfd[NPT][3];  // state of pass k-1
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int pn = j * T + tid;
      if (pn < N) {
        nm[j] = E.lump[pn] * scale;
        ninv[j] = 1.0 / nm[j];
        ncm[j] = P.damping * nm[j];
        if (pn < NFN) {
          if (is_base) {  // WarmStart::reuse from the packed state (stiffness.cpp:157)
#pragma unroll
            for (int c = 0; c < 3; ++c) u[j][c] = P.u[off + 3 * pn + c];
          } else if (P.reuse_warm) {  // probe: copy of the converged base u (:100-101)
#pragma unroll
            for (int c = 0; c < 3; ++c) u[j][c] = __ldcg(P.u + off + 3 * pn + c);
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) u[j][c] = 0.0;
          }
        } else {  // affine BC (network.cpp:254-269), Def3::apply tensor.cpp:58-62
          const double X0 = nref[j][0], X1 = nref[j][1], X2 = nref[j][2];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double fx = Fm[3 * c] * X0 + Fm[3 * c + 1] * X1 + Fm[3 * c + 2] * X2;
            u[j][c] = fx - nref[j][c];
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          vh[j][c] = 0.0;
          pu[j][c] = pv[j][c] = pa[j][c] = pf[j][c] = pfd[j][c] = 0.0;
        }
        sx[pn] = nref[j][0] + u[j][0];
        sy[pn] = nref[j][1] + u[j][1];
        sz[pn] = nref[j][2] + u[j][2];
      }
    }
    if (tid == 0) ctl.t = is_base ? P.t[p] : 0.0;
    if (LAW == 0) {
      lmin = warp_min(lmin);
      if (lane == 0) ctl.warp_min[warp] = lmin;
    }
    const bool det_ok = det3(Fm) > 0;
    __syncthreads();
    double dt_const = 0;
    if (LAW == 0) {
      double mn = INFINITY;
      for (int w = 0; w < NW; ++w) mn = smin(mn, ctl.warp_min[w]);
      dt_const = P.dt_safety * sqrt(mn);
    }

    long long k = 0;        // index of the force pass the next fiber phase evaluates
    double dt_k = 0;        // dt of iteration k (0 for the initial pass)
    double dt_last = 0;     // dt of the last committed iteration
    int status = det_ok ? FIBRA_OK : FIBRA_E_KINEMATICS;
    int conv = 0;
    long long n_done = 0;   // iterations of the returned state
    bool rewrite_fixed = false;

    while (status == FIBRA_OK) {
      // ================= fiber phase (force pass k) =================
      if (k >= 1 && warp == NW - 1) {  // decision for pass k-1 (tree-order sums)
        double sf = 0, sfix = 0;
        for (int i = lane; i < NFN; i += 32) sf += spart[i];
        for (int i = NFN + lane; i < N; i += 32) sfix += spart[i];
        sf = warp_sum(sf);
        sfix = warp_sum(sfix);
        if (lane == 0) {
          const double res = sqrt(sf);
          const double eps = P.tolerance * smax(sqrt(sfix), force_floor);
          int d = (res <= eps) ? kDecConv : 0;
          if (!isfinite(res) || !isfinite(eps)) d |= kDecExact | kDecNonfinite;
          else if (fabs(res - eps) <= 1e-10 * eps) d |= kDecExact;
          ctl.dec = d;
        }
      }
      double kmin = INFINITY;
      bool collapsed = false;
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = j * T + tid;
        if (f < M) {
          const int ia = fab[j] & 0xffff, ib = fab[j] >> 16;
          const double dx = sx[ib] - sx[ia];
          const double dy = sy[ib] - sy[ia];
          const double dz = sz[ib] - sz[ia];
          const double len = sqrt(dx * dx + dy * dy + dz * dz);
          collapsed |= (len <= fthr[j]);
          const double stretch = len / fl0[j];
          const double g = law_force<LAW>(fs[j], stretch, bo, B) / len;
          gx[f] = g * dx;
          gy[f] = g * dy;
          gz[f] = g * dz;
          if (LAW != 0) {
            const double kt = smax(fabs(law_tangent<LAW>(fs[j], stretch, bo, B)), fs[j]);
            kmin = smin(kmin, fmred[j] / kt);
          }
        }
      }
      if (collapsed) ctl.collapse = 1;
      if (LAW != 0) {
        kmin = warp_min(kmin);
        if (lane == 0) ctl.warp_min[warp] = kmin;
      }
      __syncthreads();

      // ================= node phase (pass k) =================
      if (k >= 1) {
        int d = ctl.dec;
        if (d & kDecExact) {  // reference-order norms of f_{k-1}
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int pn = j * T + tid;
            if (pn < N)
#pragma unroll
              for (int c = 0; c < 3; ++c) sx[3 * pn + c] = pf[j][c];
          }
          __syncthreads();
          if (tid < 8) {
            const int base = tid < 4 ? 0 : 3 * NFN;
            const int len = tid < 4 ? 3 * NFN : 3 * (N - NFN);
            double acc = 0;
            for (int i = tid & 3; i < len; i += 4) acc += sx[base + i] * sx[base + i];
            ctl.ex[tid] = acc;
          }
          __syncthreads();
          const double res = sqrt((ctl.ex[0] + ctl.ex[1]) + (ctl.ex[2] + ctl.ex[3]));
          const double react = sqrt((ctl.ex[4] + ctl.ex[5]) + (ctl.ex[6] + ctl.ex[7]));
          const double eps = P.tolerance * smax(react, force_floor);
          d = (res <= eps) ? kDecConv : 0;
          if (!isfinite(res)) d |= kDecNonfinite;
          rewrite_fixed = true;
          __syncthreads();  // everyone has read ctl.ex before it can be reused
        }
        if (d & kDecNonfinite) {
          status = FIBRA_E_DIVERGED;
          n_done = k - 1;
          break;
        }
        if (d & kDecConv) {
          conv = 1;
          n_done = k - 1;
          break;
        }
        if (k - 1 == P.max_iterations) {
          n_done = k - 1;
          break;
        }
        // commit iteration k
        if (!isfinite(dt_k) || !(dt_k > 0)) {
          status = FIBRA_E_BAD_DT;
          n_done = k - 1;
          break;
        }
        if (tid == 0) ctl.t += dt_k;
        dt_last = dt_k;
      }
      if (ctl.collapse) {
        status = FIBRA_E_COLLAPSE;
        n_done = k > 0 ? k - 1 : 0;
        break;
      }
      double dt_next;
      if (LAW == 0) {
        dt_next = dt_const;
      } else {
        double mn = INFINITY;
        for (int w = 0; w < NW; ++w) mn = smin(mn, ctl.warp_min[w]);
        dt_next = P.dt_safety * sqrt(mn);
      }
      const double h_k = 0.5 * dt_k;
      const double h_n = 0.5 * dt_next;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int pn = j * T + tid;
        if (pn < N) {
          double f0 = 0.0, f1 = 0.0, f2 = 0.0;  // CSR gather, ascending fiber id
          for (int i = nbeg[j]; i < nend[j]; ++i) {
            const int en = cent[i];
            const int fi = en >> 1, neg = en & 1;
            f0 = f0 + flip(gx[fi], neg);
            f1 = f1 + flip(gy[fi], neg);
            f2 = f2 + flip(gz[fi], neg);
          }
          spart[pn] = f0 * f0 + f1 * f1 + f2 * f2;
          const double fv[3] = {f0, f1, f2};
          if (pn < NFN) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double fd = ncm[j] * vh[j][c];                // kernels_scalar.cpp:15-17
              const double acc = -(fv[c] + fd) * ninv[j];
              const double vv = (k >= 1) ? vh[j][c] + h_k * acc : vh[j][c];  // relax.cpp:166
              pu[j][c] = u[j][c];
              pv[j][c] = vv;
              pa[j][c] = acc;
              pf[j][c] = fv[c];
              pfd[j][c] = fd;
              vh[j][c] = vv + h_n * acc;                          // relax.cpp:155
              u[j][c] = u[j][c] + dt_next * vh[j][c];             // relax.cpp:156
            }
            sx[pn] = nref[j][0] + u[j][0];
            sy[pn] = nref[j][1] + u[j][1];
            sz[pn] = nref[j][2] + u[j][2];
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              pu[j][c] = u[j][c];
              pf[j][c] = fv[c];
            }
            if (rewrite_fixed) {
              sx[pn] = nref[j][0] + u[j][0];
              sy[pn] = nref[j][1] + u[j][1];
              sz[pn] = nref[j][2] + u[j][2];
            }
          }
        }
      }
      rewrite_fixed = false;
      dt_k = dt_next;
      ++k;
      __syncthreads();
    }

    // ================= exit (relax.cpp:181-190, network.cpp:341-372) =================
    // Uniform across the CTA: every thread took the same break.
    __syncthreads();
    double* SF = sx;                 // f of the returned state, flat packed order (3N)
    double* SX = regB;               // x = ref + u (3N)
    double* SW = regB + 3 * nmax;    // m v^2 over free dofs (3*NFN)
    double* SE = regB + 6 * nmax;    // per-fiber strain energy (M)
    const bool zero_iter = (n_done == 0);
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int pn = j * T + tid;
      if (pn < N) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          SF[3 * pn + c] = pf[j][c];
          SX[3 * pn + c] = nref[j][c] + pu[j][c];
          if (pn < NFN) SW[3 * pn + c] = nm[j] * (pv[j][c] * pv[j][c]);
        }
      }
    }
    __syncthreads();
    if (!zero_iter && status == FIBRA_OK) {
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = j * T + tid;
        if (f < M) {  // strain_energy relax.cpp:57-72
          const int ia = fab[j] & 0xffff, ib = fab[j] >> 16;
          const double dx = SX[3 * ib] - SX[3 * ia];
          const double dy = SX[3 * ib + 1] - SX[3 * ia + 1];
          const double dz = SX[3 * ib + 2] - SX[3 * ia + 2];
          const double len = sqrt(dx * dx + dy * dy + dz * dz);
          SE[f] = law_energy<LAW>(fs[j], len / fl0[j], fl0[j], bo, B);
        }
      }
    }
    if (tid < 12) {  // reference-order reductions (4 interleaved partials)
      const int r = tid & 3, which = tid >> 2;
      const double* src = which == 0 ? SF : (which == 1 ? SF + 3 * NFN : SW);
      const int len = which == 1 ? 3 * (N - NFN) : 3 * NFN;
      double acc = 0;
      if (which < 2)
        for (int i = r; i < len; i += 4) acc += src[i] * src[i];
      else
        for (int i = r; i < len; i += 4) acc += src[i];
      ctl.ex[tid] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      SolveOut o = {};
      const double res = sqrt((ctl.ex[0] + ctl.ex[1]) + (ctl.ex[2] + ctl.ex[3]));
      const double react = sqrt((ctl.ex[4] + ctl.ex[5]) + (ctl.ex[6] + ctl.ex[7]));
      o.residual = res;
      o.eps_eff = P.tolerance * smax(react, force_floor);
      o.iterations = n_done;
      o.dt = dt_last;
      o.converged = conv;
      o.status = status;
      if (status == FIBRA_OK && !zero_iter) {
        const double ke = 0.5 * ((ctl.ex[8] + ctl.ex[9]) + (ctl.ex[10] + ctl.ex[11]));
        double se = 0;
        for (int f = 0; f < M; ++f) se += SE[f];
        o.kinetic_fraction = (ke + se) > 0 ? ke / (ke + se) : 0.0;
      }
      if (status == FIBRA_OK && conv) {  // homogenized stress + pull-back
        const double vol = det3(Fm) * box_volume;
        double sm[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int pn = NFN; pn < N; ++pn)
          for (int i = 0; i < 3; ++i)
            for (int jj = 0; jj < 3; ++jj) sm[i][jj] += SF[3 * pn + i] * SX[3 * pn + jj];
        double raw[9];
        for (int i = 0; i < 3; ++i)
          for (int jj = 0; jj < 3; ++jj) raw[3 * i + jj] = sm[i][jj] / vol;
        double asym = 0, mag = 0;
        for (int i = 0; i < 3; ++i)
          for (int jj = 0; jj < 3; ++jj) {
            asym += (raw[3 * i + jj] - raw[3 * jj + i]) * (raw[3 * i + jj] - raw[3 * jj + i]);
            mag += raw[3 * i + jj] * raw[3 * i + jj];
          }
        sym_from_full(raw, o.sigma_u);
        o.asym = mag > 0 ? sqrt(asym / mag) : 0.0;
        if (!pull_back_stress(o.sigma_u, Fm, o.pk2)) o.status = FIBRA_E_KINEMATICS;
      } else if (status == FIBRA_OK) {
        o.status = q < 0 ? FIBRA_E_NOT_CONVERGED : FIBRA_E_PROBE_FAILED;
      }
      P.out[s] = o;
      if (is_base) {
        P.t[p] = ctl.t;
        if (status == FIBRA_OK) {  // an exception leaves iters/converged untouched
          P.iters[p] += n_done;
          P.converged[p] = static_cast<unsigned char>(conv);
        }
      }
      atomicAdd(P.counters + 0, static_cast<unsigned long long>(n_done));
      atomicAdd(P.counters + 1, static_cast<unsigned long long>(n_done) * M);
      atomicAdd(P.counters + 2, static_cast<unsigned long long>(n_done) *
                                    (51ull * M + 12ull * 3 * NFN + 2ull * 3 * (N - NFN)));
      atomicAdd(P.counters + 3, 1ull);
    }
    if (is_base) {  // PackedStates writeback of the base solve (batch.cpp:169-176)
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int pn = j * T + tid;
        if (pn < N) {
          const bool fr = pn < NFN;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const long long d = off + 3 * pn + c;
            P.u[d] = pu[j][c];
            P.v[d] = fr ? pv[j][c] : 0.0;
            P.a[d] = (fr && !zero_iter) ? pa[j][c] : 0.0;
            P.f_int[d] = pf[j][c];
            P.f_damp[d] = (fr && !zero_iter) ? pfd[j][c] : 0.0;
            P.mass[d] = nm[j];
            P.inv_mass[d] = ninv[j];
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int ok = (P.out[s].status == FIBRA_OK) ? 1 : 2;
        __threadfence();
        atomicExch(P.base_flag + p, ok);
      }
    }
    __syncthreads();
  }
}

}  // namespace fibra_b200
