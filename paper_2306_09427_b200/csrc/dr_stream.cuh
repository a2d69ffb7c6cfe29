// HBM-streaming dynamic-relaxation kernel for RVEs beyond on-chip capacity: one thread-block
// cluster of C CTAs (C <= 16) solves one RVE at a time with NOTHING of the RVE resident in
// shared memory.  Per DR iteration every thread walks its nodes' incidence rows, streamed
// from HBM/L2 with coalesced 128-bit loads (step-major: lane l of warp group g reads entry
// 32 r + l of row r), gathers the other end's x from a global double buffer (pass parity),
// evaluates the fibre itself (node-centric, d' = x_other - x_own, f -= g d' from +0.0 in
// ascending fibre id -- bitwise the reference's force loop, see dr_node.cuh) and applies the
// damped update; ONE barrier.cluster (release/acquire) per iteration separates the x writes
// of pass k+1 from the x reads of pass k.  The nonlinear law adds one (the CFL minimum).
//
// Reference path (paths under /root/reference/proj): relax_solve src/relax.cpp:93-191,
// internal_forces_cfl src/network.cpp:275-324, kernels_scalar.cpp:7-65, apply_affine_bc
// network.cpp:254-269, homogenized_stress network.cpp:341-372.
//
// Cluster-wide decisions are identical in every CTA: approximate |f|^2 sums go to per-pass
// global slots (fp64 atomics; only the order of an approximate verdict's additions varies,
// and a near tie takes the exact path), collapse flags to per-pass global slots, and at a
// stop the force vector goes to a global scratch in packed order where every CTA forms the
// reference-order 4-lane sums (kernels_scalar.cpp:20-48) with one warp (fold_chain).
// Checkpoint/replay per CTA as in dr_kernel.cuh.
#pragma once

#include <cstddef>

#include "dr_cluster.cuh"
#include "dr_kernel.cuh"
#include "fastmath.cuh"

namespace fibra_b200 {

struct StreamEntryDev {     // one RveLibrary entry for dr_stream_kernel, in slot order
  int n_nodes, n_fibers, n_free_nodes, n_fix_nodes;
  int f0, node_slots, n_rows, pad0;    // node_slots = C * T * NPT (slot j*C*T + rank*T + tid)
  double max_lump, max_ea, box_volume, ea0;
  const int* slot_pn;       // [node_slots] packed node id, -1 empty
  const double* slot_ref;   // [3 node_slots]
  const double* slot_lump;  // [node_slots]
  const int* slot_deg;      // [node_slots]
  const int* group_row0;    // [node_slots / 32 + 1]
  const int* inc_x;         // [32 n_rows] x offset (in doubles) of the other end
  const double2* inc_l0;    // [32 n_rows] (l0, rcp_refined(l0)): one 128-bit load
  const double* inc_ea;     // [32 n_rows] area*modulus
  const double* inc_lump;   // [32 n_rows] lumping weight of the other end
  const int* fib_a;         // [n_fibers] packed tail (exit strain energy)
  const int* fib_b;         // [n_fibers] packed head
  const double* fib_l0;     // [n_fibers]
  const double* fib_ea;     // [n_fibers]
};

// per-cluster global scratch (doubles): X0[3S] X1[3S] SF[3N] SX[3N] SW[3NFN] SE[M]
//                                      sums[3][2] coll[3] wmin[2][C NW]
struct StreamParams {
  DrParams d;
  const StreamEntryDev* sentries;
  double* scratch;
  long long scratch_stride;  // doubles per cluster
  int s_cap, n_cap;          // slots / nodes capacity of the class (scratch layout)
  int m_cap;                 // fibres capacity
  int stage;                 // 1: this CTA's incidence rows are TMA-staged into shared
                             //    memory once per solve (they fit), 0: streamed every pass
};

// bulk copy global -> this CTA's shared memory, completing on an mbarrier (TMA engine)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(sh_addr(dst)), "l"(src), "r"(bytes), "r"(sh_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sh_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sh_addr(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(sh_addr(bar)), "r"(phase) : "memory");
}

struct __align__(16) StreamCtl {
  int solve, point, q, entry;
  int flag, skip, pad0, pad1;
  double ck_t[2], ck_dt[2];
  double ex[12];
  double t, force_floor;
  double mom[9], se;
};

// sequential sum of a[i] * b[i] (i = start + stride k) in order, one warp (fold_chain's
// shuffle scheme): the boundary moment sums of homogenized_stress (network.cpp:347-358)
__device__ __forceinline__ double fold_dot(const double* a, const double* b, int start,
                                           int stride, int count, int lane) {
  double acc = 0.0;
  for (int c0 = 0; c0 < count; c0 += 32) {
    const int i = c0 + lane;
    const double t = i < count ? __ldcg(a + start + stride * i) * __ldcg(b + start + stride * i) : 0.0;
    const int n = count - c0 < 32 ? count - c0 : 32;
    for (int s = 0; s < n; ++s) acc = acc + __shfl_sync(0xffffffffu, t, s);
  }
  return acc;
}

template <int T, int NPT, int LAWBO, bool UEA>
__global__ void __launch_bounds__(T, 1) dr_stream_kernel(StreamParams SP) {
  constexpr int LAW = LAWBO & 1;
  constexpr int bo = LAWBO >> 1;
  __shared__ StreamCtl ctl;
  __shared__ __align__(8) unsigned long long stage_bar;
  extern __shared__ __align__(16) unsigned char smem[];
  const DrParams& P = SP.d;
  constexpr int NW = T / 32;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cl_rank(), C = cl_size();
  const int CT = static_cast<int>(C) * T;  // threads of the cluster
  const int gt = static_cast<int>(rank) * T + tid;
  const unsigned ctl_sh = sh_addr(&ctl);
  double* scr = SP.scratch + static_cast<size_t>(cl_id()) * SP.scratch_stride;
  double* XG = scr;                              // [2][3 s_cap]
  double* SF = scr + 6ll * SP.s_cap;             // [3 n_cap]
  double* SX = SF + 3ll * SP.n_cap;              // [3 n_cap]
  double* SW = SX + 3ll * SP.n_cap;              // [3 n_cap]
  double* SE = SW + 3ll * SP.n_cap;              // [m_cap]
  double* SUM = SE + SP.m_cap;                   // [3][2]
  int* COLL = reinterpret_cast<int*>(SUM + 6);   // [3] (two doubles of room)
  double* WMIN = SUM + 8;                        // [2][16 NW]
  double* ckpt = P.ckpt + static_cast<size_t>(blockIdx.x) * 12 * P.ck_stride;
  const double B = P.nonlinearity;
  const long long XS = 3ll * SP.s_cap;  // doubles per x buffer

  if (tid == 0) mbar_init(&stage_bar, 1);
  unsigned stage_phase = 0;
  cl_sync();
  for (;;) {
    // ---- ticket (rank 0), broadcast into every CTA's control block ----
    if (rank == 0 && tid == 0) {
      const int t = atomicAdd(P.ticket, 1);
      int s = -1, p = 0, q = -1, flag = 0, e = 0;
      if (t < P.n_solves) {
        flag = 1;
        if (t < P.n_class) {
          p = P.order[t];
          s = p;
        } else {
          const int kk = (t - P.n_class) / 6;
          q = (t - P.n_class) % 6;
          while ((p = ld_acquire(P.done_list + kk)) < 0) __nanosleep(256);
          s = P.n_points + 6 * p + q;
          flag = ld_acquire(P.base_flag + p) == 1;
        }
        if (P.solve_skip[s]) flag = 0;
        e = P.entry_of_point[p];
        trace_start(P, s);
      }
      for (unsigned r = 0; r < C; ++r) {
        const unsigned a = cl_map(ctl_sh + offsetof(StreamCtl, solve), r);
        cl_st_s32(a, s);
        cl_st_s32(a + 4, p);
        cl_st_s32(a + 8, q);
        cl_st_s32(a + 12, e);
        cl_st_s32(a + 16, flag);
      }
    }
    cl_sync();
    const int s = ctl.solve;
    if (s < 0) break;
    const int p = ctl.point, q = ctl.q, e = ctl.entry;
    if (!ctl.flag) {
      if (rank == 0 && tid == 0) {
        SolveOut o = {};
        o.status = P.solve_skip[s] ? P.solve_skip[s] : FIBRA_E_NOT_CONVERGED;
        P.out[s] = o;
        trace_end(P, s, 0);
        if (q < 0) publish_base(P, p, 2);
      }
      cl_sync();
      continue;
    }
    const StreamEntryDev& E = SP.sentries[e];
    const double scale = P.density_scale / E.max_lump;  // setup_mass relax.cpp:35-43
    const int F0 = E.f0;
    const double s_uni = P.ea_scale * E.ea0;
    int deg[NPT], row0[NPT], nsteps[NPT], slot[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      slot[j] = j * CT + gt;
      deg[j] = E.slot_deg[slot[j]];
      row0[j] = E.group_row0[slot[j] >> 5];
      nsteps[j] = E.group_row0[(slot[j] >> 5) + 1] - row0[j];
    }
#define NREF(j, c) __ldg(E.slot_ref + 3 * slot[j] + (c))
    // this CTA's incidence rows: block j holds the rows of its warp groups for slot block j
    // (contiguous in HBM); staged = one TMA bulk copy per array and block into shared
    // memory, once per solve
    const int* rIX[NPT];
    const double2* rIL[NPT];
    const double* rIE[NPT];
    const double* rIM[NPT];
    int rbase[NPT];
    {
      unsigned char* sp = smem;
      unsigned total = 0;
      size_t e0s[NPT], nes[NPT];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int g0 = (j * CT + static_cast<int>(rank) * T) >> 5;
        rbase[j] = E.group_row0[g0];
        const int rows = E.group_row0[g0 + NW] - rbase[j];
        const size_t e0 = 32ull * rbase[j], ne = 32ull * rows;
        e0s[j] = e0;
        nes[j] = ne;
        if (SP.stage) {
          int* sx = reinterpret_cast<int*>(sp);
          double2* sl = reinterpret_cast<double2*>(sx + ne);
          double* se = reinterpret_cast<double*>(sl + ne);
          double* sm = se + (UEA ? 0 : ne);
          total += static_cast<unsigned>(ne * (4 + 16 + (UEA ? 0 : 8) + (LAW != 0 ? 8 : 0)));
          rIX[j] = sx;
          rIL[j] = sl;
          rIE[j] = se;
          rIM[j] = sm;
          sp = reinterpret_cast<unsigned char*>(sm + (LAW != 0 ? ne : 0));
        } else {
          rIX[j] = E.inc_x + e0;
          rIL[j] = E.inc_l0 + e0;
          rIE[j] = E.inc_ea + e0;
          rIM[j] = E.inc_lump + e0;
        }
      }
      if (SP.stage && tid == 0) {
        // the previous solve's generic-proxy reads of these bytes are ordered before the
        // bulk (async-proxy) writes; then arm the barrier and issue the copies
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&stage_bar, total);  // the single arrival of this phase
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
          if (!nes[j]) continue;
          const unsigned ne = static_cast<unsigned>(nes[j]);
          bulk_g2s(const_cast<int*>(rIX[j]), E.inc_x + e0s[j], 4u * ne, &stage_bar);
          bulk_g2s(const_cast<double2*>(rIL[j]), E.inc_l0 + e0s[j], 16u * ne, &stage_bar);
          if (!UEA) bulk_g2s(const_cast<double*>(rIE[j]), E.inc_ea + e0s[j], 8u * ne, &stage_bar);
          if (LAW != 0) bulk_g2s(const_cast<double*>(rIM[j]), E.inc_lump + e0s[j], 8u * ne, &stage_bar);
        }
      }
    }

    // ---- per-solve setup (relax.cpp:95-145) ----
    double Fm[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fm[i] = P.solve_F[9 * s + i];
    const long long off = P.offsets[p];
    const bool is_base = q < 0;
    double u[NPT][3], vh[NPT][3], ninv[NPT], ncm[NPT], mj[NPT];
    double lmin = INFINITY;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int sl = slot[j];
      const int pn = E.slot_pn[sl];
      const double m = E.slot_lump[sl] * scale;
      mj[j] = m;
      ninv[j] = 1.0 / m;
      ncm[j] = P.damping * m;
      if (LAW == 0)  // the CFL bound of the linear law (reduced_mass_l0 relax.cpp:46-55)
        for (int st = 0; st < deg[j]; ++st) {
          const int ix = 32 * (row0[j] + st) + (sl & 31);
          const double mb = E.inc_lump[ix] * scale;
          const double mred = m * mb / (m + mb) * E.inc_l0[ix].x;
          const double sj = UEA ? s_uni : P.ea_scale * E.inc_ea[ix];
          lmin = smin(lmin, mred / smax(fabs(law_tangent<0>(sj, 1.0, 0, B)), sj));
        }
      if (sl < F0) {
        if (pn < 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) u[j][c] = 0.0;
        } else if (is_base) {  // WarmStart::reuse (stiffness.cpp:157)
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
        const double X0r = NREF(j, 0), X1r = NREF(j, 1), X2r = NREF(j, 2);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double fx = Fm[3 * c] * X0r + Fm[3 * c + 1] * X1r + Fm[3 * c + 2] * X2r;
          u[j][c] = fx - NREF(j, c);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) vh[j][c] = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double xc = NREF(j, c) + u[j][c];
        XG[3ll * sl + c] = xc;
        if (sl >= F0) XG[XS + 3ll * sl + c] = xc;  // fixed nodes never move: both buffers
      }
      if (sl < F0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ckpt[c * P.ck_stride + j * T + tid] = u[j][c];
          ckpt[(3 + c) * P.ck_stride + j * T + tid] = 0.0;
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
    if (rank == 0 && tid < 6) SUM[tid] = 0.0;
    if (rank == 0 && tid < 3) COLL[tid] = 0;
    if (LAW == 0) {
      lmin = warp_min(lmin);
      if (lane == 0) WMIN[rank * NW + warp] = lmin;
    }
    const bool det_ok = det3(Fm) > 0;
    if (SP.stage) {  // the rows of this solve have landed
      mbar_wait(&stage_bar, stage_phase);
      stage_phase ^= 1;
    }
    cl_sync();
    double dt_const = 0;
    if (LAW == 0) {
      double mn = INFINITY;
      for (int w = 0; w < static_cast<int>(C) * NW; ++w) mn = smin(mn, __ldcg(WMIN + w));
      dt_const = P.dt_safety * sqrt(mn);
    }
    cl_sync();  // WMIN read everywhere before any pass writes it

    int k = 0, target = -1, status = det_ok ? FIBRA_OK : FIBRA_E_KINEMATICS, conv = 0;
    double dt_k = 0;
    bool rewrite_fixed = false;
    double fk[NPT][3];
    while (status == FIBRA_OK) {
      // ---- verdict of pass k-1 (identical in every CTA) ----
      if (target < 0 && k >= 1) {
        const int sp = (k - 1) % 3;
        if (__ldcg(COLL + sp)) {  // network.cpp:291 throws inside the force pass of k-1
          status = FIBRA_E_COLLAPSE;
          k -= 1;
          break;
        }
        const double res = sqrt(__ldcg(SUM + 2 * sp));
        const double eps = P.tolerance * smax(sqrt(__ldcg(SUM + 2 * sp + 1)), ctl.force_floor);
        int d = (res <= eps) ? kDecConv : 0;
        if (!isfinite(res) || !isfinite(eps)) d |= kDecExact | kDecNonfinite;
        else if (fabs(res - eps) <= 1e-10 * eps) d |= kDecExact;
        if (k - 1 <= ctl.skip) d = 0;
        if ((d & (kDecConv | kDecExact)) || k - 1 == P.max_iterations) {
          target = k - 1;
          k = target / kCkInterval * kCkInterval;  // newest checkpoint <= target
          const int b = (k / kCkInterval) & 1;
          dt_k = ctl.ck_dt[b];
          const double* ck = ckpt + b * 6 * P.ck_stride;
          double* Xk = XG + (k & 1) * XS;
#pragma unroll
          for (int j = 0; j < NPT; ++j)
            if (slot[j] < F0)
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                u[j][c] = __ldcg(ck + c * P.ck_stride + j * T + tid);
                vh[j][c] = __ldcg(ck + (3 + c) * P.ck_stride + j * T + tid);
                Xk[3ll * slot[j] + c] = NREF(j, c) + u[j][c];
              }
          cl_sync();  // every CTA has read the slots of pass k-1
          if (tid == 0) ctl.t = ctl.ck_t[b];
          if (rank == 0 && tid < 6) SUM[tid] = 0.0;
          if (rank == 0 && tid < 3) COLL[tid] = 0;
          rewrite_fixed = false;
          cl_sync();
          continue;
        }
      }
      if (k >= 1) {  // commit iteration k (relax.cpp:150-153)
        if (!isfinite(dt_k) || !(dt_k > 0)) {
          status = FIBRA_E_BAD_DT;
          break;
        }
        if (tid == 0) ctl.t += dt_k;
      }
      if (rank == 0 && tid < 3) {  // the slot of pass k+1 (last read at the start of k-1)
        const int sn = (k + 1) % 3;
        if (tid < 2) SUM[2 * sn + tid] = 0.0;
        if (tid == 2) COLL[sn] = 0;
      }

      // ================= forces of pass k (incidence rows streamed) =================
      const double* Xc = XG + (k & 1) * XS;
      bool collapsed = false;
      double kmin = INFINITY;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const double x0 = NREF(j, 0) + u[j][0];
        const double x1 = NREF(j, 1) + u[j][1];
        const double x2 = NREF(j, 2) + u[j][2];
        double f0 = 0.0, f1 = 0.0, f2 = 0.0;
        const int n_j = deg[j], ns = nsteps[j];
        struct Inc {
          double dx, dy, dz, len, g, l0;
          bool ok;
        };
        auto eval = [&](int st) {
          Inc r;
          const int ix = 32 * (row0[j] - rbase[j] + st) + lane;  // within this CTA's block
          const int xo = SP.stage ? rIX[j][ix] : __ldg(rIX[j] + ix);
          const double2 lr = SP.stage ? rIL[j][ix] : __ldg(rIL[j] + ix);  // 128-bit coalesced
          r.dx = __ldcg(Xc + xo) - x0;  // d' = x_other - x_own
          r.dy = __ldcg(Xc + xo + 1) - x1;
          r.dz = __ldcg(Xc + xo + 2) - x2;
          r.l0 = lr.x;
          const double sj = UEA ? s_uni : P.ea_scale * (SP.stage ? rIE[j][ix] : __ldg(rIE[j] + ix));
          bool o1, o2, o3 = true;
          r.len = sqrt_fast(r.dx * r.dx + r.dy * r.dy + r.dz * r.dz, o1);
          const double stretch = div_fast_rcp(r.len, lr.x, lr.y, o2);
          if (LAW == 0) {
            r.g = div_fast(law_force<0>(sj, stretch, bo, B), r.len, o3);
          } else {
            r.g = law_force<LAW>(sj, stretch, bo, B) / r.len;
            if (st < n_j) {
              const double mb = (SP.stage ? rIM[j][ix] : __ldg(rIM[j] + ix)) * scale;
              const double mred = mj[j] * mb / (mj[j] + mb) * lr.x;  // relax.cpp:50-53
              const double kt = smax(fabs(law_tangent<LAW>(sj, stretch, bo, B)), sj);
              kmin = smin(kmin, mred / kt);
            }
          }
          r.ok = (o1 && o2 && o3) || st >= n_j;
          return r;
        };
        auto slow = [&](Inc& r, int st) {
          if (!r.ok) {
            const int ix = 32 * (row0[j] - rbase[j] + st) + lane;
            const double sj = UEA ? s_uni : P.ea_scale * (SP.stage ? rIE[j][ix] : __ldg(rIE[j] + ix));
            r.len = sqrt(r.dx * r.dx + r.dy * r.dy + r.dz * r.dz);
            r.g = law_force<LAW>(sj, r.len / r.l0, bo, B) / r.len;
          }
        };
        auto add = [&](const Inc& r, int st) {  // f_tail -= g d; f_head += g d
          if (st < n_j) {
            collapsed |= (r.len <= 1e-8 * r.l0);  // network.cpp:291
            f0 = f0 - r.g * r.dx;
            f1 = f1 - r.g * r.dy;
            f2 = f2 - r.g * r.dz;
          }
        };
        int st = 0;
        for (; st + 1 < ns; st += 2) {
          Inc a = eval(st), b = eval(st + 1);
          if (__any_sync(0xffffffffu, !(a.ok && b.ok))) {
            slow(a, st);
            slow(b, st + 1);
          }
          add(a, st);
          add(b, st + 1);
        }
        if (st < ns) {
          Inc a = eval(st);
          if (__any_sync(0xffffffffu, !a.ok)) slow(a, st);
          add(a, st);
        }
        fk[j][0] = f0;
        fk[j][1] = f1;
        fk[j][2] = f2;
        const double part = warp_sum(f0 * f0 + f1 * f1 + f2 * f2);
        if (lane == 0) atomicAdd(SUM + 2 * (k % 3) + (slot[j] < F0 ? 0 : 1), part);
      }
      if (collapsed) atomicExch(COLL + k % 3, 1);
      if (LAW != 0) {
        kmin = warp_min(kmin);
        if (lane == 0) WMIN[(k & 1) * 16 * NW + rank * NW + warp] = kmin;
        cl_sync();  // dt of iteration k+1 = CFL minimum over all fibres of pass k
      }

      const double h_k = 0.5 * dt_k;
      if (k == target) {
        // ---- exact verdict at the target pass: reference-order norms in every CTA ----
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
          const int pn = E.slot_pn[slot[j]];
          if (pn >= 0)
#pragma unroll
            for (int c = 0; c < 3; ++c) SF[3 * pn + c] = fk[j][c];
        }
        cl_sync();
        if (warp == 0) {
          const int NFN = E.n_free_nodes, NFIX = E.n_fix_nodes;
          for (int r = 0; r < 8; ++r) {
            const int base = r < 4 ? 0 : 3 * NFN, len = r < 4 ? 3 * NFN : 3 * NFIX;
            const int cnt = len > (r & 3) ? (len - (r & 3) + 3) / 4 : 0;
            const double v = fold_chain<true>(SF, base + (r & 3), 4, cnt, lane);
            if (lane == 0) ctl.ex[r] = v;
          }
        }
        __syncthreads();
        const double res = sqrt((ctl.ex[0] + ctl.ex[1]) + (ctl.ex[2] + ctl.ex[3]));
        const double react = sqrt((ctl.ex[4] + ctl.ex[5]) + (ctl.ex[6] + ctl.ex[7]));
        const double eps = P.tolerance * smax(react, ctl.force_floor);
        __syncthreads();
        const bool nonfinite = k >= 1 && !isfinite(res);
        conv = res <= eps;
        if (nonfinite || conv || k == P.max_iterations) {
          if (nonfinite) {
            status = FIBRA_E_DIVERGED;
            break;
          }
          const bool base_solve = ctl.q < 0;
          const long long soff = P.offsets[ctl.point];
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int sl = slot[j];
            const int pn = E.slot_pn[sl];
            if (pn < 0) continue;
            const double m = E.slot_lump[sl] * scale;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double fd = 0.0, acc = 0.0, vv = 0.0;
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
        if (tid == 0) ctl.skip = target;
        target = -1;
        rewrite_fixed = true;
        cl_sync();  // SF read everywhere before a later stop rewrites it
      }
      // ---- damped update + speculative half step / drift of iteration k+1 ----
      double dt_next;
      if (LAW == 0) {
        dt_next = dt_const;
      } else {
        double mn = INFINITY;
        for (int w = 0; w < static_cast<int>(C) * NW; ++w)
          mn = smin(mn, __ldcg(WMIN + (k & 1) * 16 * NW + w));
        dt_next = P.dt_safety * sqrt(mn);
      }
      const double h_n = 0.5 * dt_next;
      const bool save = target < 0 && ((k + 1) % kCkInterval == 0);
      const int sb = ((k + 1) / kCkInterval) & 1;
      double* Xn = XG + ((k + 1) & 1) * XS;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = slot[j];
        if (sl < F0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double fd = ncm[j] * vh[j][c];              // kernels_scalar.cpp:15-17
            const double acc = -(fk[j][c] + fd) * ninv[j];
            const double vv = (k >= 1) ? vh[j][c] + h_k * acc : vh[j][c];  // relax.cpp:166
            vh[j][c] = vv + h_n * acc;                          // relax.cpp:155
            u[j][c] = u[j][c] + dt_next * vh[j][c];             // relax.cpp:156
            Xn[3ll * sl + c] = NREF(j, c) + u[j][c];
          }
          if (save) {
            double* ck = ckpt + sb * 6 * P.ck_stride;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              ck[c * P.ck_stride + j * T + tid] = u[j][c];
              ck[(3 + c) * P.ck_stride + j * T + tid] = vh[j][c];
            }
          }
        } else if (rewrite_fixed) {
#pragma unroll
          for (int c = 0; c < 3; ++c) Xn[3ll * sl + c] = NREF(j, c) + u[j][c];
        }
      }
      rewrite_fixed = false;
      cl_sync();
      if (save && tid == 0) {
        ctl.ck_t[sb] = ctl.t;
        ctl.ck_dt[sb] = dt_next;
      }
      dt_k = dt_next;
      ++k;
    }

    // ================= exit (relax.cpp:181-190, network.cpp:341-372) =================
    const int n_done = (status == FIBRA_OK) ? k : (k > 0 ? k - 1 : 0);
    const bool zero_iter = (n_done == 0);
    const int N = E.n_nodes, M = E.n_fibers, NFN = E.n_free_nodes, NFIX = E.n_fix_nodes;
    const int s_ = ctl.solve, p_ = ctl.point;
    const bool base_solve = ctl.q < 0;
    // every CTA leaves the loop at the same pass with the same status
    cl_sync();
    if (status == FIBRA_OK && !zero_iter)
      for (int f = gt; f < M; f += CT) {  // strain_energy relax.cpp:57-72
        const int ta = E.fib_a[f], hb = E.fib_b[f];
        const double dx = __ldcg(SX + 3 * hb) - __ldcg(SX + 3 * ta);
        const double dy = __ldcg(SX + 3 * hb + 1) - __ldcg(SX + 3 * ta + 1);
        const double dz = __ldcg(SX + 3 * hb + 2) - __ldcg(SX + 3 * ta + 2);
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        const double l0 = E.fib_l0[f];
        const double sj = UEA ? s_uni : P.ea_scale * E.fib_ea[f];
        SE[f] = law_energy<LAW>(sj, len / l0, l0, bo, B);
      }
    cl_sync();
    if (rank == 0 && status == FIBRA_OK && warp < 3) {  // reference-order reductions
      if (warp == 0) {
        for (int r = 0; r < 12; ++r) {
          const int which = r >> 2, rr = r & 3;
          const double* src = which == 0 ? SF : (which == 1 ? SF + 3 * NFN : SW);
          const int len = which == 1 ? 3 * NFIX : 3 * NFN;
          const int cnt = len > rr ? (len - rr + 3) / 4 : 0;
          const double v = which < 2 ? fold_chain<true>(src, rr, 4, cnt, lane)
                                     : fold_chain<false>(src, rr, 4, cnt, lane);
          if (lane == 0) ctl.ex[r] = v;
        }
      } else if (warp == 1) {
        const double v = zero_iter ? 0.0 : fold_chain<false>(SE, 0, 1, M, lane);
        if (lane == 0) ctl.se = v;
      } else if (conv) {  // homogenized_stress moment sums, boundary nodes ascending
        for (int i = 0; i < 3; ++i)
          for (int jj = 0; jj < 3; ++jj) {
            const double v = fold_dot(SF + i, SX + jj, 3 * NFN, 3, N - NFN, lane);
            if (lane == 0) ctl.mom[3 * i + jj] = v;
          }
      }
    }
    __syncthreads();
    if (rank == 0 && tid == 0) {
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
          const double se = ctl.se;
          o.kinetic_fraction = (ke + se) > 0 ? ke / (ke + se) : 0.0;
        }
        if (conv) {
          for (int i = 0; i < 9; ++i) o.moment[i] = ctl.mom[i];
          o.box_volume = E.box_volume;
        } else {
          o.status = base_solve ? FIBRA_E_NOT_CONVERGED : FIBRA_E_PROBE_FAILED;
        }
      }
      P.out[s_] = o;
      trace_end(P, s_, n_done);
      if (base_solve) {
        P.t[p_] = ctl.t;
        if (status == FIBRA_OK) {
          P.iters[p_] += n_done;
          P.converged[p_] = static_cast<unsigned char>(conv);
        } else {
          P.converged[p_] = 0;
        }
      }
      atomicAdd(P.counters + 0, static_cast<unsigned long long>(n_done));
      atomicAdd(P.counters + 1, static_cast<unsigned long long>(n_done) * M);
      atomicAdd(P.counters + 2, static_cast<unsigned long long>(n_done) *
                                    (51ull * M + 12ull * 3 * NFN + 2ull * 3 * NFIX));
      atomicAdd(P.counters + 3, 1ull);
      atomicAdd(P.counters + 4, static_cast<unsigned long long>(n_done) *
                                    (28ull * M + 12ull * 3 * NFN + 2ull * 3 * NFIX));
    }
    if (base_solve) {
      __threadfence();
      cl_sync();  // every CTA's PackedStates writes precede the publication
      if (rank == 0 && tid == 0) publish_base(P, p_, P.out[s_].status == FIBRA_OK ? 1 : 2);
    }
    cl_sync();
#undef NREF
  }
}

}  // namespace fibra_b200
