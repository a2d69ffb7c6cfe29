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
// Bitwise contract with the reference: --fmad=false, IEEE div/sqrt
// (fastmath.cuh replays nvcc's own sequences); x = ref + u rounded per node; each node's
// force is accumulated from +0.0 over its incident fibers in ascending fiber id (CSR, no
// atomics), reproducing f[a] -= g*d / f[b] += g*d of network.cpp:298-303; the damped update
// follows kernels_scalar.cpp:15-17 and relax.cpp:155-166 literally.
//
// Per DR iteration the CTA runs two phases separated by __syncthreads():
//   fiber phase: each thread evaluates FPT register-resident fibers, reading x records
//                (24-byte AoS) from shared memory and writing one g*d record each;
//   node phase:  each thread owns NPT nodes (u and the half-step velocity in registers),
//                gathers its CSR list, applies the damped central-difference update and
//                writes the next x record.
// Slots are placed by host/schedule.cpp so the random gathers are (mostly) bank-conflict
// free; empty fiber/node slots hold harmless dummies so the hot loop has no per-slot
// branches.  CSR lists are padded to even length with a record of +0.0 (f + 0.0 == f for
// every f the accumulation can produce, since it starts at +0.0 and never reaches -0.0).
// Each fiber writes one +g*d record; its tail node reads it back as fma(-1, r, f), which
// equals f - r (one rounding, the product is exact).
// The convergence test is off the critical path: node threads store one |f|^2 per slot
// (two buffers by pass parity); at the end of the next node phase the last warp -- the
// lightest gather, fixed nodes -- reduces them with a short branch-free tree and compares
// in squares, and the node phase after that reads the verdict, two iterations late
// (FIBRA_DECIDER_NODE=0: in the last warp's fiber phase, one late).  Every warp owns
// fibers; a warp whose last fiber row is empty skips it.  The CTA keeps two
// checkpoints of (u, v_half, t, dt) in global memory; when a verdict says "stop at k"
// (converged, iteration cap, non-finite, or a near tie |R - eps| <= 1e-10 eps where the
// tree sum could disagree with the reference's 4-lane sum) it restores the newest
// checkpoint at or before k, replays to k -- bit-identical, the arithmetic is
// deterministic -- and decides at k with the reference-order sums.
#pragma once

#include <cstdint>
#include <type_traits>

#include "fastmath.cuh"
#include "fibra_cuda.h"
#include "libm_glibc.cuh"
#include "tensor.cuh"

namespace fibra_b200 {

struct EntryDev {          // one RveLibrary entry in HBM, already in slot order
  int n_nodes, n_fibers, n_free_nodes, n_fix_nodes;
  int f0, node_slots, fiber_slots, gd_slots;  // gd_slots includes dummies + zero record
  int thread_slots, max_pairs, pad1, pad2;    // NPT*T (32 dummy x records follow)
  double max_lump, max_ea, box_volume, pad3;
  const int* slot_pn;      // [thread_slots] packed node id per slot, -1 empty
  const double* slot_ref;  // [3*thread_slots] reference coordinates by slot
  const double* slot_lump; // [thread_slots] lumping weight by slot (1 when empty)
  const int* csr_npairs;   // [thread_slots] CSR entry pairs per slot (lists padded to even)
  const int2* csr_pairs;   // [max_pairs][thread_slots] step-major: lanes read consecutive
                           // pairs; entry = 24*gslot | (node is the stored tail) << 31
  const int* fib_ab;       // [fiber_slots] 24*tail_slot | 24*head_slot << 16
  const int* fib_g;        // [fiber_slots] 24*gslot: the fiber's +g*d record
  const int* fib_id;       // [fiber_slots] reference fiber id, -1 dummy
  const double* fib_l0;    // [fiber_slots]
  const double* fib_ea;    // [fiber_slots] area*modulus
};

struct SolveOut {          // one DR solve (base or probe)
  double moment[9];        // sum over boundary nodes of r_i x_j (network.cpp:347-358)
  double box_volume;
  long long iterations;
  double residual, eps_eff, kinetic_fraction, dt;
  int converged;
  int status;
};

struct NodeEntryDev;  // dr_node.cuh

struct DrParams {
  const EntryDev* entries;
  const NodeEntryDev* nentries;  // node-centric kernel (dr_node.cuh)
  const int* entry_of_point;
  const long long* offsets;
  double *u, *v, *a, *f_int, *f_damp, *mass, *inv_mass, *t;
  long long* iters;
  unsigned char* converged;
  const double* solve_F;       // 9 per solve
  const int* solve_skip;       // nonzero: solve pre-failed by prep (status code)
  SolveOut* out;
  int* base_flag;              // per point: 0 pending, 1 converged, 2 failed
  const int* order;            // base ticket -> point (longest expected solve first)
  int* done_list;              // points in base-completion order (-1: not yet)
  int* ticket;                 // [0] next ticket, [1] done_list fill count
  int first_wave_sms;          // > 0: the grid is two blocks per SM over this many SMs
  unsigned long long* counters;  // [0] iterations [1] fiber-iterations [2] pipe ops [3] solves
                                 // [4] algorithmic flops
  double* ckpt;                // [grid][2][6][ck_stride]
  int ck_stride, ck_interval;
  int n_points;                // all bound points (solve index layout)
  int n_class, n_solves;       // this launch: points of its kernel class, their solves
  int x_bytes, g_bytes, part_slots, csr_cap;  // shared-memory layout capacities
  int reuse_warm;
  int law_buckling_off;
  double ea_scale, nonlinearity;
  double damping, tolerance, dt_safety, density_scale;
  long long max_iterations;
  unsigned long long* phase_prof;  // optional [grid][NW][8] cycle accumulators
  unsigned long long* trace;       // optional [solve][4]: start ns, end ns,
                                   // sm << 32 | class << 24 | block, iterations (FIBRA_TRACE)
  int trace_class;
  int shared_queue;                // several launches share this class's ticket counter:
                                   // every ticket comes from it (no first-wave dealing)
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_start(const DrParams& P, int s) {
  if (P.trace) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    P.trace[4 * s] = global_ns();
    P.trace[4 * s + 2] = (static_cast<unsigned long long>(sm) << 32) |
                         (static_cast<unsigned long long>(P.trace_class) << 24) | blockIdx.x;
  }
}

__device__ __forceinline__ void trace_end(const DrParams& P, int s, long long iters) {
  if (P.trace) {
    P.trace[4 * s + 1] = global_ns();
    P.trace[4 * s + 3] = static_cast<unsigned long long>(iters);
  }
}

enum : int { kDecConv = 1, kDecExact = 2, kDecNonfinite = 4 };

// Checkpoints of (u, v_half) are taken at resume passes 0, C, 2C, ... alternating between
// two buffers (buffer (r/C)&1 holds resume pass r); a stop detected one pass late replays
// at most 2C passes.
constexpr int kCkInterval = 8;

// Diagnostics switches for layout experiments (defaults are the product configuration):
// FIBRA_TOPO_REG 1 keeps each fiber's x-record offsets, record offset and rest length in
// registers for the whole solve, 0 re-reads them from L1 every fiber phase.
#ifndef FIBRA_TOPO_REG
#define FIBRA_TOPO_REG 1
#endif
// FIBRA_DECIDER_NODE 1: the last warp decides pass k-1 at the end of node phase k (its
// gather is the lightest) and node phase k+1 reads it; 0: it decides in fiber phase k and
// node phase k reads it.
#ifndef FIBRA_DECIDER_NODE
#define FIBRA_DECIDER_NODE 1
#endif
constexpr int kLag = FIBRA_DECIDER_NODE ? 2 : 1;
#ifndef FIBRA_GATHER_AHEAD  // how many steps ahead the gather loads its CSR pair (1 or 2)
#define FIBRA_GATHER_AHEAD 1
#endif  // node phase k reads the verdict of k-kLag

// Per-warp phase cycle counters, compiled only into the diagnostics build
// (FIBRA_PHASE_PROF=1 python -m paper_2306_09427_b200.build -> lib/libfibra_b200_prof.so).
#ifdef FIBRA_PHASE_PROF
#define FB_PROF(...) __VA_ARGS__
#else
#define FB_PROF(...)
#endif

struct __align__(16) DrCtl {
  int solve, point, q, entry;
  int flag, collapse, skip;  // skip: last pass whose exact verdict said "continue"
  int dec[2];                // speculative verdict of pass r in dec[r & 1] (decider warp)
  double ck_t[2], ck_dt[2];  // checkpoint buffers: t after, dt of, the resume pass
  double warp_min[32];
  double ex[12];
  double t;
  double force_floor;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// a finished base solve publishes its flag, then its point in the completion FIFO from
// which probe tickets are served
__device__ __forceinline__ void publish_base(const DrParams& P, int p, int flag) {
  __threadfence();
  atomicExch(P.base_flag + p, flag);
  st_release(P.done_list + atomicAdd(P.ticket + 1, 1), p);
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

// +1.0 or -1.0 by the CSR entry's bit 31: fma(sign_one(e), r, f) == f + r or f - r, one
// rounding (the product is exact) -- the gather's signed add in one LOP3 + one DFMA
__device__ __forceinline__ double sign_one(int entry) {
  return __hiloint2double((entry & static_cast<int>(0x80000000u)) | 0x3ff00000, 0);
}


template <class Tp>
__device__ __forceinline__ Tp* sm_at(unsigned char* base, int byte_off) {
  return reinterpret_cast<Tp*>(base + byte_off);
}

// axial force N(lambda) and tangent (network.cpp:16-38); s = ea_scale*ea.  expm1 / exp are
// the host libm's own operation sequences (libm_glibc.cuh), so the exponential law is
// bitwise too.
template <int LAW>
__device__ __forceinline__ double law_force(double s, double stretch, int buckling_off,
                                            double B) {
  if (LAW == 0) return (buckling_off && stretch < 1.0) ? 0.0 : s * (stretch - 1.0);
  if (buckling_off && stretch < 1.0) return 0.0;
  return s / B * glibc::expm1(B * (stretch - 1.0));
}

template <int LAW>
__device__ __forceinline__ double law_tangent(double s, double stretch, int buckling_off,
                                              double B) {
  if (buckling_off && stretch < 1.0) return 0.0;
  if (LAW == 0) return s;
  return s * glibc::exp(B * (stretch - 1.0));
}

template <int LAW>
__device__ __forceinline__ double law_energy(double s, double stretch, double rl,
                                             int buckling_off, double B) {  // :40-53
  if (buckling_off && stretch < 1.0) return 0.0;
  const double e = stretch - 1.0;
  if (LAW == 0) return 0.5 * s * rl * e * e;
  return rl * s / B * (glibc::expm1(B * e) / B - e);
}

// UEA: every fiber of the library has the same area*modulus (true for generated
// networks), so the axial stiffness s = ea_scale*EA is one scalar instead of FPT registers.
template <int T, int FPT, int NPT, int LAWBO, int MINB, bool UEA>
__global__ void __launch_bounds__(T, MINB) dr_persistent_kernel(DrParams P) {
  // LAWBO = law (0 linear, 1 exponential) + 2 * buckling_off: compile-time law flavour
  constexpr int LAW = LAWBO & 1;
  constexpr int bo = LAWBO >> 1;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ DrCtl ctl;
  constexpr int NW = T / 32;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // shared layout: [X: x records (24 B/slot) | exact scratch][G: g*d records | exit scratch]
  //                [SPART: |f|^2 per node slot][CSR entries]
  unsigned char* X = smem;
  unsigned char* G = smem + P.x_bytes;
  double* spart = reinterpret_cast<double*>(G + P.g_bytes);  // [kLag][NPT * T]
  int2* cent = reinterpret_cast<int2*>(spart + kLag * NPT * T);  // step-major CSR pairs
  double* ckpt = P.ckpt + static_cast<size_t>(blockIdx.x) * 12 * P.ck_stride;

  const double B = P.nonlinearity;

  // register-resident topology of the loaded entry
  // (x-record offsets, record offset and rest length are re-read from L1 each fiber phase:
  //  kept in registers they would be live through the node phase's gather, whose loads
  //  then cannot be issued ahead of their uses under the 2-CTA/SM register budget)
  double frl0[FPT], fs[FPT], fmred[FPT];  // frl0: rcp_refined(l0), loop invariant
#if FIBRA_TOPO_REG
  int fab_r[FPT], fgo_r[FPT];
  double fl0_r[FPT];
#endif
  int npair[NPT];
  int frows = FPT;  // fiber rows holding a real fiber in some lane of this warp
  double ninv[NPT], ncm[NPT];  // (reference coordinates: NREF, read through L1 when used)
  int cur_entry = -1;
  bool first_ticket = true;
  double s_uni = 0;  // UEA: the common ea_scale*EA
#define SJ(j) (UEA ? s_uni : fs[j])
#define NREF(j, c) __ldg(E.slot_ref + 3 * ((j) * T + tid) + (c))

  for (;;) {
    // Tickets [0, nc) are the base solves of this kernel class in P.order; tickets
    // [nc, 7nc) are probes, served in the order base solves finish (six per finished base),
    // so a CTA only waits for a base when every finished base's probes are already taken.
    // Solve index: base p -> p, probe q of p -> n + 6p + q (the layout post_kernel reads);
    // -1 = queue drained.  The first wave is dealt by block index: the block scheduler puts
    // blocks [0, #SM) one per SM and blocks [#SM, 2 #SM) in the second slots, so SM j runs
    // tickets j and 2 #SM - 1 - j -- the longest expected solve next to the shortest of
    // the wave, and two of the longest never share an SM; later tickets come from the
    // counter.
    if (tid == 0) {
      int t;
      if (P.shared_queue) {
        t = atomicAdd(P.ticket, 1);
      } else if (first_ticket) {
        const int b = static_cast<int>(blockIdx.x), m = P.first_wave_sms;
        t = (m > 0 && b >= m) ? 3 * m - 1 - b : b;
      } else {
        t = static_cast<int>(gridDim.x) + atomicAdd(P.ticket, 1);
      }
      first_ticket = false;
      int s = -1;
      if (t < P.n_solves) {
        int p, q = -1, flag = 1;
        if (t < P.n_class) {
          p = P.order[t];
          s = p;
        } else {
          const int k = (t - P.n_class) / 6;
          q = (t - P.n_class) % 6;
          while ((p = ld_acquire(P.done_list + k)) < 0) __nanosleep(256);
          s = P.n_points + 6 * p + q;
          flag = ld_acquire(P.base_flag + p) == 1;
        }
        if (P.solve_skip[s]) flag = 0;
        ctl.point = p;
        ctl.q = q;
        ctl.entry = P.entry_of_point[p];
        ctl.collapse = 0;
        ctl.flag = flag;
        trace_start(P, s);
      }
      ctl.solve = s;
    }
    __syncthreads();
    const int s = ctl.solve;
    if (s < 0) break;
    const int p = ctl.point, q = ctl.q, e = ctl.entry;
    if (!ctl.flag) {  // pre-failed (prep) or base failed: nothing to solve
      if (tid == 0) {
        SolveOut o = {};
        o.status = P.solve_skip[s] ? P.solve_skip[s] : FIBRA_E_NOT_CONVERGED;
        P.out[s] = o;
        trace_end(P, s, 0);
        if (q < 0) publish_base(P, p, 2);
      }
      __syncthreads();
      continue;
    }

    const EntryDev& E = P.entries[e];
    const double scale = P.density_scale / E.max_lump;  // setup_mass relax.cpp:35-43
    // sizes are re-read from E where needed: keeping them live across the DR loop costs
    // registers the 2-CTA/SM budget does not have
    const int F0 = E.f0;
    if (e != cur_entry) {
      cur_entry = e;
      s_uni = P.ea_scale * E.fib_ea[0];
      for (int i = tid; i < (E.max_pairs + 2) * E.thread_slots; i += T) cent[i] = E.csr_pairs[i];
      // dummy x records for empty fiber slots (16 tails (0,0,0), 16 heads (1,0,0)), and the
      // zero g*d record (last record)
      if (tid < 96) sm_at<double>(X, 24 * E.thread_slots)[tid] = (tid >= 48 && tid % 3 == 0) ? 1.0 : 0.0;
      if (tid < 3) sm_at<double>(G, 24 * (E.gd_slots - 1))[tid] = 0.0;
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = j * T + tid;
        {  // (NaN outside [2^-900, 2^1000]: the fast-path range test then sends the fiber
           //  to the built-in operators, fastmath.cuh fiber_fast_ok)
          const double l0 = E.fib_l0[f];
          frl0[j] = (l0 >= 0x1p-900 && l0 <= 0x1p1000) ? rcp_refined(l0) : __longlong_as_double(0x7ff8000000000000ll);
        }
#if FIBRA_TOPO_REG
        fab_r[j] = E.fib_ab[f];
        fgo_r[j] = E.fib_g[f];
        fl0_r[j] = E.fib_l0[f];
#endif
        if (!UEA) fs[j] = P.ea_scale * E.fib_ea[f];
      }
      int rows = 0;
#pragma unroll
      for (int j = 0; j < FPT; ++j)
        if (E.fib_id[j * T + tid] >= 0) rows = j + 1;
      frows = __reduce_max_sync(0xffffffffu, rows);
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        npair[j] = E.csr_npairs[sl];
      }
    }
    // ---- per-solve setup (relax.cpp:95-145) ----
    double Fm[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fm[i] = P.solve_F[9 * s + i];
    const long long off = P.offsets[p];
    const bool is_base = q < 0;
    double lmin = INFINITY;
#pragma unroll
    for (int j = 0; j < FPT; ++j) {  // reduced_mass_l0 relax.cpp:46-55
      const int fab = E.fib_ab[j * T + tid];
      const int ta = (fab & 0xffff) / 24, hb = (static_cast<unsigned>(fab) >> 16) / 24;
      if (ta < E.thread_slots) {
        const double ma = E.slot_lump[ta] * scale;
        const double mb = E.slot_lump[hb] * scale;
        fmred[j] = ma * mb / (ma + mb) * E.fib_l0[j * T + tid];
      } else {
        fmred[j] = INFINITY;  // dummy fiber
      }
      if (LAW == 0) {  // linear: the CFL bound is stretch independent
        const double kt = smax(fabs(law_tangent<0>(SJ(j), 1.0, 0, B)), SJ(j));
        lmin = smin(lmin, fmred[j] / kt);
      }
    }
    double u[NPT][3], vh[NPT][3];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int sl = j * T + tid;
      const int pn = E.slot_pn[sl];
      const double m = E.slot_lump[sl] * scale;
      ninv[j] = 1.0 / m;
      ncm[j] = P.damping * m;
      if (sl < F0) {
        if (pn < 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) u[j][c] = 0.0;
        } else if (is_base) {  // WarmStart::reuse from the packed state (stiffness.cpp:157)
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
        const double X0 = NREF(j, 0), X1 = NREF(j, 1), X2 = NREF(j, 2);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double fx = Fm[3 * c] * X0 + Fm[3 * c + 1] * X1 + Fm[3 * c + 2] * X2;
          u[j][c] = fx - NREF(j, c);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) vh[j][c] = 0.0;
      double* xr = sm_at<double>(X, 24 * sl);
      xr[0] = NREF(j, 0) + u[j][0];
      xr[1] = NREF(j, 1) + u[j][1];
      xr[2] = NREF(j, 2) + u[j][2];
      if (sl < F0) {  // checkpoint "resume at pass 0": u_0, v = 0
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ckpt[c * P.ck_stride + sl] = u[j][c];
          ckpt[(3 + c) * P.ck_stride + sl] = 0.0;
        }
      }
    }
    if (tid == 0) {
      ctl.t = is_base ? P.t[p] : 0.0;
      ctl.ck_t[0] = ctl.t;
      ctl.ck_dt[0] = 0.0;
      ctl.force_floor = P.ea_scale * E.max_ea * 1e-12;  // relax.cpp:112
      ctl.skip = -1;
    }
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

    int k = 0;              // force pass the next fiber phase evaluates
    int target = -1;        // pass at which to stop and decide exactly (replay mode)
    double dt_k = 0;        // dt of iteration k (0 for the initial pass)
    int status = det_ok ? FIBRA_OK : FIBRA_E_KINEMATICS;
    int conv = 0;
    bool rewrite_fixed = false;

    // fiber | bar1 | node: verdict/commit checks | gather | exact + update + decider | bar2
    FB_PROF(long long pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0, pc4 = 0, pc5 = 0, tq = 0;)
    while (status == FIBRA_OK) {
      // ================= fiber phase (force pass k) =================
      FB_PROF(tq = clock64());
      // Speculative verdict of pass r by the last warp.  Lane l sums slots l, l+32, ...:
      // row i = slot/32 is free iff i < F0/32.  Loads first, then a tree: a short chain
      // (any summation order will do).
      auto decide = [&](int r) {
        constexpr int R = NPT * T / 32;
        const int R0 = F0 >> 5;
        const double* sp = spart + (r % kLag) * (NPT * T);
        double vf[R], vx[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const double v = sp[32 * i + lane];
          vf[i] = i < R0 ? v : 0.0;
          vx[i] = i < R0 ? 0.0 : v;
        }
#pragma unroll
        for (int w = 1; w < R; w *= 2)
#pragma unroll
          for (int i = 0; i + w < R; i += 2 * w) {
            vf[i] += vf[i + w];
            vx[i] += vx[i + w];
          }
        double sf = vf[0], sfix = vx[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sf += __shfl_xor_sync(0xffffffffu, sf, o);
          sfix += __shfl_xor_sync(0xffffffffu, sfix, o);
        }
        // squared form of res <= tol * max(sqrt(sfix), floor); a near tie (|res - eps| <=
        // 1e-10 eps, within ~2e-10 in squares) or a tiny threshold is decided exactly with
        // the reference's sums; a pass already decided exactly ("continue" at a near tie)
        // is not re-decided
        if (lane == 0) {
          const double fl = ctl.force_floor;
          const double e2 = (P.tolerance * P.tolerance) * smax(sfix, fl * fl);
          int d = (sf <= e2) ? kDecConv : 0;
          if (!isfinite(sf) || !isfinite(e2)) d |= kDecExact | kDecNonfinite;
          else if (fabs(sf - e2) <= 4e-10 * e2 || e2 < 0x1p-900) d |= kDecExact;
          ctl.dec[r & 1] = (r > ctl.skip) ? d : 0;
        }
      };
      if (!FIBRA_DECIDER_NODE && target < 0 && k >= 1 && warp == NW - 1) decide(k - 1);
      {
        double kmin = INFINITY;
        bool collapsed = false;
        // fibres in blocks of <= 4 so only one block's temporaries are live (the FPT >= 6
        // shapes spill otherwise); FPT <= 3 is a single block, the unchanged config-2 code
        auto fiber_block = [&](auto j0c, auto j1c) {
          constexpr int J0 = decltype(j0c)::value, J1 = decltype(j1c)::value;
          bool fast = true;
          double dx[J1 - J0], dy[J1 - J0], dz[J1 - J0], g[J1 - J0], fl0[J1 - J0];
          int fgo[J1 - J0];
#pragma unroll
          for (int jj = 0; jj < J1 - J0; ++jj) {
            const int j = J0 + jj;
#if FIBRA_TOPO_REG
            const int fab = fab_r[j];
            fgo[jj] = fgo_r[j];
            fl0[jj] = fl0_r[j];
#else
            const int fab = E.fib_ab[j * T + tid];
            fgo[jj] = E.fib_g[j * T + tid];
            fl0[jj] = E.fib_l0[j * T + tid];
#endif
            const double* xa_ = sm_at<double>(X, fab & 0xffff);
            const double* xb_ = sm_at<double>(X, static_cast<unsigned>(fab) >> 16);
            dx[jj] = xb_[0] - xa_[0];
            dy[jj] = xb_[1] - xa_[1];
            dz[jj] = xb_[2] - xa_[2];
            bool o1, o2 = true, o3 = true;
            const double len = sqrt_fast(dx[jj] * dx[jj] + dy[jj] * dy[jj] + dz[jj] * dz[jj], o1);
            collapsed |= (len <= 1e-8 * fl0[jj]);  // network.cpp:291
            if (LAW == 0) {  // one range test for both divisions (fastmath.cuh)
              const double stretch = div_rcp_raw(len, fl0[jj], frl0[j]);
              const double n = law_force<0>(SJ(j), stretch, bo, B);
              g[jj] = div_rcp_raw(n, len, rcp_refined(len));
              o2 = fiber_fast_ok(len, stretch, n);
            } else {
              const double stretch = div_fast_rcp(len, fl0[jj], frl0[j], o2);
              g[jj] = law_force<LAW>(SJ(j), stretch, bo, B) / len;
              const double kt = smax(fabs(law_tangent<LAW>(SJ(j), stretch, bo, B)), SJ(j));
              kmin = smin(kmin, fmred[j] / kt);
            }
            fast = fast && o1 && o2 && o3;
          }
          if (!__all_sync(0xffffffffu, fast)) {  // rare: special operands -> built-in ops
#pragma unroll
            for (int jj = 0; jj < J1 - J0; ++jj) {
              const int j = J0 + jj;
              const double len = sqrt(dx[jj] * dx[jj] + dy[jj] * dy[jj] + dz[jj] * dz[jj]);
              collapsed |= (len <= 1e-8 * fl0[jj]);  // exact length (e.g. 0): network.cpp:291
              const double stretch = len / fl0[jj];
              g[jj] = law_force<LAW>(SJ(j), stretch, bo, B) / len;
            }
          }
#pragma unroll
          for (int jj = 0; jj < J1 - J0; ++jj) {  // one record +g*d (the tail gathers -1 *)
            const int j = J0 + jj;
            double* gr = sm_at<double>(G, fgo[jj]);
            gr[0] = g[jj] * dx[jj];
            gr[1] = g[jj] * dy[jj];
            gr[2] = g[jj] * dz[jj];
          }
        };
#ifdef FIBRA_FIBER_B1  // diagnostics: fibers per block of the first block
        constexpr int B1 = FIBRA_FIBER_B1 < FPT ? FIBRA_FIBER_B1 : FPT;
#else
        constexpr int B1 = FPT < 4 ? FPT : (FPT + 1) / 2;
#endif
        if constexpr (B1 < FPT) {
          fiber_block(std::integral_constant<int, 0>(), std::integral_constant<int, B1>());
          if (frows > B1)
            fiber_block(std::integral_constant<int, B1>(), std::integral_constant<int, FPT>());
        } else if constexpr (FPT >= 2) {
          if (frows == FPT)
            fiber_block(std::integral_constant<int, 0>(), std::integral_constant<int, FPT>());
          else  // the warp's last fiber row is empty
            fiber_block(std::integral_constant<int, 0>(), std::integral_constant<int, FPT - 1>());
        } else {
          fiber_block(std::integral_constant<int, 0>(), std::integral_constant<int, FPT>());
        }
        if (collapsed) ctl.collapse = 1;
        if (LAW != 0) {
          kmin = warp_min(kmin);
          if (lane == 0) ctl.warp_min[warp] = kmin;
        }
      }
      FB_PROF({ const long long t1 = clock64(); pc0 += t1 - tq; tq = t1; })
      __syncthreads();
      FB_PROF({ const long long t1 = clock64(); pc1 += t1 - tq; tq = t1; })

      // ================= node phase (pass k) =================
      if (target < 0 && k >= kLag) {
        const int dec = ctl.dec[(k - kLag) & 1];
        if ((dec & (kDecConv | kDecExact)) || k - kLag == P.max_iterations) {
          // stop at k-kLag: replay from the newest checkpoint that resumes at or before it
          target = k - kLag;
          // resume points are the multiples of kCkInterval, alternating between buffers;
          // the newest one <= target is still held (the saves at target+1 .. target+kLag --
          // at most one of them, kCkInterval > kLag -- used the other)
          k = target / kCkInterval * kCkInterval;
          const int b = (k / kCkInterval) & 1;
          dt_k = ctl.ck_dt[b];
          const double* ck = ckpt + b * 6 * P.ck_stride;
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int sl = j * T + tid;
            if (sl < F0) {
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                u[j][c] = __ldcg(ck + c * P.ck_stride + sl);
                vh[j][c] = __ldcg(ck + (3 + c) * P.ck_stride + sl);
              }
            }
            double* xr = sm_at<double>(X, 24 * sl);
            xr[0] = NREF(j, 0) + u[j][0];
            xr[1] = NREF(j, 1) + u[j][1];
            xr[2] = NREF(j, 2) + u[j][2];
          }
          if (tid == 0) {
            ctl.t = ctl.ck_t[b];
            ctl.collapse = 0;
          }
          rewrite_fixed = false;
          __syncthreads();
          // verdicts of passes before the replay are void (every read of them is done)
          if (FIBRA_DECIDER_NODE && tid == 0) ctl.dec[0] = ctl.dec[1] = 0;
          continue;
        }
      }
      // the last warp decides pass k-1 at the end of this phase (not at an exact pass)
      const bool decide_here = FIBRA_DECIDER_NODE && target < 0 && k >= 1 && warp == NW - 1;
      if (k >= 1) {  // commit iteration k (relax.cpp:150-153)
        if (!isfinite(dt_k) || !(dt_k > 0)) {
          status = FIBRA_E_BAD_DT;
          break;
        }
        if (tid == 0) ctl.t += dt_k;
      }
      if (ctl.collapse) {
        status = FIBRA_E_COLLAPSE;
        break;
      }
      const double h_k = 0.5 * dt_k;
      FB_PROF({ const long long t1 = clock64(); pc4 += t1 - tq; tq = t1; })
      double fk[NPT][3];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        double f0 = 0.0, f1 = 0.0, f2 = 0.0;  // CSR gather, ascending fiber id
        // the next step's pair is loaded one step ahead (row max_pairs is padding), so a
        // step's six record loads depend only on registers and issue back to back
        int2 ep = cent[sl];
#if FIBRA_GATHER_AHEAD == 2  // diagnostics: the pair two steps ahead (two padding rows)
        int2 ep1 = cent[NPT * T + sl];
#endif
        // not unrolled: with the CSR pair loaded a step ahead, ptxas's default 4-way unroll
        // only adds register pressure (2.39 -> 2.33 us per CTA-iteration without it);
        // FIBRA_GATHER_UNROLL=n (diagnostics) sets another factor
#ifndef FIBRA_GATHER_UNROLL
#define FIBRA_GATHER_UNROLL 1
#endif
#define FB_PRAGMA(x) _Pragma(#x)
#define FB_UNROLL(n) FB_PRAGMA(unroll n)
        FB_UNROLL(FIBRA_GATHER_UNROLL)
        for (int kp = 0; kp < npair[j]; ++kp) {  // two incidences per step
          const int2 en = cent[(kp + FIBRA_GATHER_AHEAD) * (NPT * T) + sl];
          const double* g0 = sm_at<double>(G, ep.x & 0x7fffffff);  // the fiber's +g*d
          const double* g1 = sm_at<double>(G, ep.y & 0x7fffffff);
          const double a0 = g0[0], a1 = g0[1], a2 = g0[2];
          const double b0 = g1[0], b1 = g1[1], b2 = g1[2];
          const double sa = sign_one(ep.x), sb = sign_one(ep.y);  // -1 for the tail
          // f -= g*d for the tail, f += g*d for the head (network.cpp:298-303)
          f0 = __fma_rn(sa, a0, f0);
          f1 = __fma_rn(sa, a1, f1);
          f2 = __fma_rn(sa, a2, f2);
          f0 = __fma_rn(sb, b0, f0);
          f1 = __fma_rn(sb, b1, f1);
          f2 = __fma_rn(sb, b2, f2);
#if FIBRA_GATHER_AHEAD == 2
          ep = ep1;
          ep1 = en;
#else
          ep = en;
#endif
        }
        fk[j][0] = f0;
        fk[j][1] = f1;
        fk[j][2] = f2;
        const double q = f0 * f0 + f1 * f1 + f2 * f2;
        spart[(k % kLag) * (NPT * T) + sl] = q;
      }
      FB_PROF({ const long long t1 = clock64(); pc5 += t1 - tq; tq = t1; })
      if (k == target) {
        // ---- exact verdict at the target pass (reference-order norms) ----
        double* SF = reinterpret_cast<double*>(X);
        __syncthreads();  // every x read of this pass is done; SF reuses X
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
          const int pn = E.slot_pn[j * T + tid];
          if (pn >= 0)
#pragma unroll
            for (int c = 0; c < 3; ++c) SF[3 * pn + c] = fk[j][c];
        }
        __syncthreads();
        if (tid < 8) {
          const int NFN = E.n_free_nodes, NFIX = E.n_fix_nodes;
          const int base = tid < 4 ? 0 : 3 * NFN;
          const int len = tid < 4 ? 3 * NFN : 3 * NFIX;
          double acc = 0;
          for (int i = tid & 3; i < len; i += 4) acc += SF[base + i] * SF[base + i];
          ctl.ex[tid] = acc;
        }
        __syncthreads();
        const double res = sqrt((ctl.ex[0] + ctl.ex[1]) + (ctl.ex[2] + ctl.ex[3]));
        const double react = sqrt((ctl.ex[4] + ctl.ex[5]) + (ctl.ex[6] + ctl.ex[7]));
        const double eps = P.tolerance * smax(react, ctl.force_floor);
        __syncthreads();  // ctl.ex consumed before anyone reuses it
        const bool nonfinite = k >= 1 && !isfinite(res);
        conv = res <= eps;
        if (nonfinite || conv || k == P.max_iterations) {
          if (nonfinite) {
            status = FIBRA_E_DIVERGED;
            break;
          }
          // Final state of iteration k, written straight to the exit scratch (SF already
          // holds f) and, for base solves, to the PackedStates (batch.cpp:169-176).  Doing
          // it here keeps no exit arrays alive across the DR loop.
          double* SX = reinterpret_cast<double*>(G);
          double* SW = SX + 3 * E.n_nodes;
          const bool base_solve = ctl.q < 0;
          const long long soff = P.offsets[ctl.point];
          const double mscale = P.density_scale / E.max_lump;
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int sl = j * T + tid;
            const int pn = E.slot_pn[sl];
            if (pn < 0) continue;
            const double m = E.slot_lump[sl] * mscale;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double fd = 0.0, acc = 0.0, vv = 0.0;  // fixed dofs / 0-iteration exit
              if (sl < F0 && k >= 1) {
                fd = ncm[j] * vh[j][c];                // kernels_scalar.cpp:15-17
                acc = -(fk[j][c] + fd) * ninv[j];
                vv = vh[j][c] + h_k * acc;             // relax.cpp:166
              }
              SX[3 * pn + c] = NREF(j, c) + u[j][c];
              if (sl < F0) SW[3 * pn + c] = m * (vv * vv);
              if (base_solve) {
                const long long d = soff + 3 * pn + c;
                P.u[d] = u[j][c];
                P.v[d] = vv;
                P.a[d] = acc;
                P.f_int[d] = fk[j][c];
                P.f_damp[d] = fd;
                P.mass[d] = m;
                P.inv_mass[d] = ninv[j];
              }
            }
          }
          break;
        }
        if (tid == 0) ctl.skip = target;  // near tie that did not stop: continue normally
        target = -1;
        rewrite_fixed = true;
      }
      // ---- damped update + speculative half step / drift of iteration k+1 ----
      double dt_next;
      if (LAW == 0) {
        dt_next = dt_const;
      } else {
        double mn = INFINITY;
        for (int w = 0; w < NW; ++w) mn = smin(mn, ctl.warp_min[w]);
        dt_next = P.dt_safety * sqrt(mn);
      }
      const double h_n = 0.5 * dt_next;
      const bool save = target < 0 && ((k + 1) % kCkInterval == 0);
      const int sb = ((k + 1) / kCkInterval) & 1;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        double* xr = sm_at<double>(X, 24 * sl);
        if (sl < F0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double fd = ncm[j] * vh[j][c];              // kernels_scalar.cpp:15-17
            const double acc = -(fk[j][c] + fd) * ninv[j];
            const double vv = (k >= 1) ? vh[j][c] + h_k * acc : vh[j][c];  // relax.cpp:166
            vh[j][c] = vv + h_n * acc;                          // relax.cpp:155
            u[j][c] = u[j][c] + dt_next * vh[j][c];             // relax.cpp:156
          }
          xr[0] = NREF(j, 0) + u[j][0];
          xr[1] = NREF(j, 1) + u[j][1];
          xr[2] = NREF(j, 2) + u[j][2];
          if (save) {
            double* ck = ckpt + sb * 6 * P.ck_stride;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              ck[c * P.ck_stride + sl] = u[j][c];
              ck[(3 + c) * P.ck_stride + sl] = vh[j][c];
            }
          }
        } else if (rewrite_fixed) {
          xr[0] = NREF(j, 0) + u[j][0];
          xr[1] = NREF(j, 1) + u[j][1];
          xr[2] = NREF(j, 2) + u[j][2];
        }
      }
      rewrite_fixed = false;
      if (decide_here) decide(k - 1);
      FB_PROF({ const long long t1 = clock64(); pc2 += t1 - tq; tq = t1; })
      __syncthreads();
      FB_PROF({ const long long t1 = clock64(); pc3 += t1 - tq; tq = t1; })
      if (save && tid == 0) {
        ctl.ck_t[sb] = ctl.t;
        ctl.ck_dt[sb] = dt_next;
      }
      dt_k = dt_next;
      ++k;
    }

    // ================= exit (relax.cpp:181-190, network.cpp:341-372) =================
    // Uniform across the CTA.  On a normal stop k == target and the final state of
    // iteration k is already in the exit scratch / PackedStates; solver errors skip all
    // of it (the reference leaves a partially updated state behind on a throw).
    const int n_done = (status == FIBRA_OK) ? k : (k > 0 ? k - 1 : 0);
    FB_PROF(if (P.phase_prof && lane == 0) {
      unsigned long long* pp = P.phase_prof + (static_cast<size_t>(blockIdx.x) * NW + warp) * 8;
      pp[0] += pc0; pp[1] += pc1; pp[2] += pc4; pp[3] += pc5; pp[4] += pc2; pp[5] += pc3;
    })
    const bool zero_iter = (n_done == 0);
    const int N = E.n_nodes, M = E.n_fibers, NFN = E.n_free_nodes, NFIX = E.n_fix_nodes;
    const int s_ = ctl.solve, p_ = ctl.point;
    const bool base_solve = ctl.q < 0;
    __syncthreads();
    double* SF = reinterpret_cast<double*>(X);                 // f, flat packed order (3N)
    double* SX = reinterpret_cast<double*>(G);                 // x = ref + u (3N)
    double* SW = SX + 3 * N;                                   // m v^2, free dofs (3*NFN)
    double* SE = SW + 3 * NFN;                                 // strain energy per fiber (M)
    if (status == FIBRA_OK && !zero_iter) {
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = E.fib_id[j * T + tid];
        if (f >= 0) {  // strain_energy relax.cpp:57-72 (reference fiber id order)
          const int fab = E.fib_ab[j * T + tid];
          const int ta = E.slot_pn[(fab & 0xffff) / 24];
          const int hb = E.slot_pn[(static_cast<unsigned>(fab) >> 16) / 24];
          const double dx = SX[3 * hb] - SX[3 * ta];
          const double dy = SX[3 * hb + 1] - SX[3 * ta + 1];
          const double dz = SX[3 * hb + 2] - SX[3 * ta + 2];
          const double len = sqrt(dx * dx + dy * dy + dz * dz);
          const double l0 = E.fib_l0[j * T + tid];
          SE[f] = law_energy<LAW>(SJ(j), len / l0, l0, bo, B);
        }
      }
    }
    if (status == FIBRA_OK && tid < 12) {  // reference-order reductions (4 partials)
      const int r = tid & 3, which = tid >> 2;
      const double* src = which == 0 ? SF : (which == 1 ? SF + 3 * NFN : SW);
      const int len = which == 1 ? 3 * NFIX : 3 * NFN;
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
      o.iterations = n_done;
      o.status = status;
      if (status == FIBRA_OK) {
        const double res = sqrt((ctl.ex[0] + ctl.ex[1]) + (ctl.ex[2] + ctl.ex[3]));
        const double react = sqrt((ctl.ex[4] + ctl.ex[5]) + (ctl.ex[6] + ctl.ex[7]));
        o.residual = res;
        o.eps_eff = P.tolerance * smax(react, ctl.force_floor);
        o.dt = zero_iter ? 0.0 : dt_k;
        o.converged = conv;
        if (!zero_iter) {
          const double ke = 0.5 * ((ctl.ex[8] + ctl.ex[9]) + (ctl.ex[10] + ctl.ex[11]));
          double se = 0;
          for (int f = 0; f < M; ++f) se += SE[f];
          o.kinetic_fraction = (ke + se) > 0 ? ke / (ke + se) : 0.0;
        }
        if (conv) {  // homogenized_stress moment sums, boundary nodes ascending
          // (network.cpp:347-358); the division by J V, symmetrization and pull-back run in
          // post_kernel so their register footprint stays out of this kernel
          double sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
          for (int pn = NFN; pn < N; ++pn) {
            const double r0 = SF[3 * pn], r1 = SF[3 * pn + 1], r2 = SF[3 * pn + 2];
            const double x0 = SX[3 * pn], x1 = SX[3 * pn + 1], x2 = SX[3 * pn + 2];
            sm[0] += r0 * x0; sm[1] += r0 * x1; sm[2] += r0 * x2;
            sm[3] += r1 * x0; sm[4] += r1 * x1; sm[5] += r1 * x2;
            sm[6] += r2 * x0; sm[7] += r2 * x1; sm[8] += r2 * x2;
          }
          for (int i = 0; i < 9; ++i) o.moment[i] = sm[i];
          o.box_volume = E.box_volume;
        } else {
          o.status = base_solve ? FIBRA_E_NOT_CONVERGED : FIBRA_E_PROBE_FAILED;
        }
      }
      P.out[s_] = o;
      trace_end(P, s_, n_done);
      if (base_solve) {
        P.t[p_] = ctl.t;
        if (status == FIBRA_OK) {  // a throw leaves iters untouched (relax.cpp:187)
          P.iters[p_] += n_done;
          P.converged[p_] = static_cast<unsigned char>(conv);
        } else {
          P.converged[p_] = 0;     // apply_affine_bc already cleared it (network.cpp:268)
        }
      }
      atomicAdd(P.counters + 0, static_cast<unsigned long long>(n_done));
      atomicAdd(P.counters + 1, static_cast<unsigned long long>(n_done) * M);
      atomicAdd(P.counters + 2, static_cast<unsigned long long>(n_done) *
                                    (51ull * M + 12ull * 3 * NFN + 2ull * 3 * NFIX));
      atomicAdd(P.counters + 3, 1ull);
      atomicAdd(P.counters + 4, static_cast<unsigned long long>(n_done) *  // F_alg
                                    (28ull * M + 12ull * 3 * NFN + 2ull * 3 * NFIX));
    }
    if (base_solve) {
      // every thread wrote part of the converged u its probes warm-start from: each one
      // fences its own stores before thread 0 publishes
      __threadfence();
      __syncthreads();
      if (tid == 0) publish_base(P, p_, P.out[s_].status == FIBRA_OK ? 1 : 2);
    }
    __syncthreads();
  }
#undef SJ
#undef NREF
}

}  // namespace fibra_b200
