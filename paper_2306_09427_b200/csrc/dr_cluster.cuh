// Cluster dynamic-relaxation kernel: one thread-block cluster of C CTAs solves one large
// RVE at a time (RVEs that do not fit one CTA's shared memory; configs 3 and 4).
//
// Same reference path and the same bitwise contract as dr_kernel.cuh (relax.cpp:93-191,
// network.cpp:254-372, kernels_scalar.cpp:7-65).  The RVE is split by
// host/cluster_schedule.cpp; per DR iteration every CTA runs
//   fiber phase: its owned fibers read x of their tail (own node) and head (own node or a
//                halo copy) from local shared memory, store +g*d into their local record
//                and, if the head lives in another CTA, into that CTA's record
//                (st.shared::cluster);
//   barrier.cluster
//   node phase:  its nodes gather their CSR lists from local records (tail incidences
//                negated through the entry's sign bit, ascending fiber id), apply the damped
//                update, write x locally and push it to the halo slots of the CTAs that read
//                it;
//   barrier.cluster
// Cluster-wide quantities stay exact and use no DSMEM atomics (64-bit shared-memory min is a
// CAS emulation that is not atomic against another CTA's remote access): every warp pushes
// its CFL minimum into its own slot in every CTA and each warp takes the min over all slots
// (order independent); the convergence verdict is formed from
// per-CTA partial sums that every CTA pushes to every CTA, so all CTAs take the identical
// decision two passes late; at a stop the force vector goes to a per-cluster global
// scratch in packed order and each CTA evaluates the reference-order 4-lane sums
// (kernels_scalar.cpp:34-48) itself.  Checkpoint/replay is per CTA as in dr_kernel.cuh.
#pragma once

#include <cstddef>
#include <type_traits>

#include "dr_kernel.cuh"

namespace fibra_b200 {

struct PartDev {            // one CTA's share of one RVE
  int f0, node_slots, halo, max_pairs;
  int max_push, n_records, pad0, pad1;
  const int* slot_pn;       // [TS] packed node id, -1 empty
  const double* slot_ref;   // [3 TS]
  const double* slot_lump;  // [TS]
  const int* csr_npairs;    // [TS]
  const int2* csr_pairs;    // [max_pairs][TS] byte offset of a local record | 1u<<31 negate
  const int* push_n;        // [TS] halo copies of this slot's x
  const int* push_dst;      // [max_push][TS] rank << 16 | byte offset of the halo x record
  const int* fib_ab;        // [FS] x byte offsets: tail | head << 16 (own or halo slot)
  const int* fib_gt;        // [FS] byte offset of the fiber's local record (= 24*(j*(T-32)+tid))
  const int* fib_gh;        // [FS] rank << 24 | byte offset of its record in the head's CTA, -1
  const int* fib_id;        // [FS] reference fiber id, -1 dummy
  const double* fib_l0;     // [FS]
  const double* fib_ea;     // [FS]
  const double* fib_lt;     // [FS] lumping weight of the tail node
  const double* fib_lh;     // [FS] lumping weight of the head node
};

struct ClusterEntryDev {
  int n_nodes, n_fibers, n_free_nodes, n_fix_nodes;
  double max_lump, max_ea, box_volume, ea0;
  const PartDev* parts;     // [C]
  int mirror;               // cross fibers evaluated by both CTAs (host/cluster_schedule.hpp)
  int pad;
};

struct ClusterParams {
  DrParams d;
  const ClusterEntryDev* centries;
  double* scratch;          // per cluster: SF[3N] | SX[3N] | SW[3 NFN] | SE[M]
  long long scratch_stride;
  int push_cap;             // push_dst ints staged in shared memory
  int halo_stride;          // bytes between the two halo banks (mirror mode)
  int debug_no_local;       // diagnostics: cluster barrier for the fiber -> node handoff too
  int pad;
};

struct __align__(16) ClusterCtl {
  int solve, point, q, entry;
  int flag, dec, skip, pad0;  // skip: last pass whose exact verdict said "continue"
  int collapse[2], pad1[2];   // [pass & 1]: a fiber of that pass collapsed somewhere
  double ck_t[2], ck_dt[2];
  double ex[12];
  double se, mom[9];          // exit: strain energy and boundary moment sums (rank 0)
  double t, force_floor;
  double part[2][16][2];       // [pass & 1][rank] partial |f|^2 (free, fixed)
  double wmin[16 * 16];        // [rank * NW + warp] CFL minima of every warp of the cluster
};

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// barrier.cluster with release/acquire (SASS: MEMBAR.ALL.GPU + UCGABAR_ARV/WAIT + CCTL.IVALL);
// a relaxed arrive would save ~0.2 us per barrier but gives DSMEM stores no ordering
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ unsigned sh_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cl_map(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st_f64(unsigned a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st_s32(unsigned a, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Reference-order sequential sum of src[start + stride*i], i = 0..count-1 (squared terms for
// SQ: `acc += v * v`, kernels_scalar.cpp), by one warp: lanes load 32 consecutive terms (the
// next 32 in flight), then every lane folds them in order through shuffles -- the same
// additions in the same order as one thread's loop, without its serial L2 round trips.
template <bool SQ>
__device__ __forceinline__ double fold_chain(const double* src, int start, int stride, int count,
                                             int lane) {
  double acc = 0.0;
  double v = lane < count ? __ldcg(src + start + stride * lane) : 0.0;
  for (int c0 = 0; c0 < count; c0 += 32) {
    const int nx = c0 + 32 + lane;
    const double vn = nx < count ? __ldcg(src + start + stride * nx) : 0.0;
    const double t = SQ ? v * v : v;
    const int n = count - c0;
    if (n >= 32) {
#pragma unroll
      for (int s = 0; s < 32; ++s) acc = acc + __shfl_sync(0xffffffffu, t, s);
    } else {
      for (int s = 0; s < n; ++s) acc = acc + __shfl_sync(0xffffffffu, t, s);
    }
    v = vn;
  }
  return acc;
}

// min over the n cluster-wide warp slots, evaluated by one warp (every lane gets it)
__device__ __forceinline__ double slots_min(const double* w, int n, int lane) {
  double m = INFINITY;
  for (int i = lane; i < n; i += 32) m = smin(m, w[i]);
  return warp_min(m);
}

template <int T, int FPT, int NPT, int LAWBO, bool UEA>
__global__ void __launch_bounds__(T, 1) dr_cluster_kernel(ClusterParams CP) {
  // LAWBO = law (0 linear, 1 exponential) + 2 * buckling_off: compile-time law flavour
  constexpr int LAW = LAWBO & 1;
  constexpr int bo = LAWBO >> 1;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ ClusterCtl ctl;
  const DrParams& P = CP.d;
  constexpr int NW = T / 32;
  static_assert(NW <= 16, "ClusterCtl::wmin holds 16 warps per CTA");
  constexpr int TS = NPT * T;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cl_rank(), C = cl_size();

  // shared layout: [X: own slots | 2 dummy | halo bank 0 | halo bank 1][G: records][SPART]
  //                [CSR pairs][push list]
  unsigned char* X = smem;
  unsigned char* G = smem + P.x_bytes;
  double* spart = reinterpret_cast<double*>(G + P.g_bytes);
  int2* cent = reinterpret_cast<int2*>(spart + TS);
  int* pushd = reinterpret_cast<int*>(cent + P.csr_cap);
  double* ckpt = P.ckpt + static_cast<size_t>(blockIdx.x) * 12 * P.ck_stride;
  double* scr = CP.scratch + static_cast<size_t>(cl_id()) * CP.scratch_stride;
  const unsigned X_sh = sh_addr(X), G_sh = sh_addr(G), ctl_sh = sh_addr(&ctl);
  const unsigned off_solve = offsetof(ClusterCtl, solve), off_collapse = offsetof(ClusterCtl, collapse);
  // fiber -> node handoff: a CTA barrier when every gathered record is written locally
  // (mirror mode) and dt needs no cluster-wide minimum (linear law), else a cluster barrier
  const unsigned off_part = offsetof(ClusterCtl, part);
  const unsigned off_wmin = offsetof(ClusterCtl, wmin) + 8 * (rank * NW + warp);  // my warp's slot
  // push this warp's CFL minimum into its slot of every CTA (lane r -> CTA r)
  auto push_wmin = [&](double v) {
    if (lane < static_cast<int>(C)) cl_st_f64(cl_map(ctl_sh + off_wmin, lane), v);
  };

  const double B = P.nonlinearity;

  int fab[FPT], fgh[FPT];
  double fl0[FPT], frl0[FPT], fs[FPT], fmred[FPT];  // frl0: rcp_refined(l0), loop invariant
  int npair[NPT], npush[NPT];
  double nref[NPT][3], ninv[NPT], ncm[NPT];
  int cur_entry = -1;
  double s_uni = 0;
#define SJ(j) (UEA ? s_uni : fs[j])

  cl_sync();  // every CTA of the cluster is running before any DSMEM access

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
        const unsigned a = cl_map(ctl_sh + off_solve, r);
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

    const ClusterEntryDev& E = CP.centries[e];
    const PartDev& Q = E.parts[rank];
    const bool local_handoff = LAW == 0 && E.mirror && !CP.debug_no_local;
    // With a CTA barrier only between the phases, a neighbour may already push x of pass
    // k+1 while this CTA still reads the halo of pass k: halo copies are double-buffered by
    // pass parity (it cannot get two passes ahead: the cluster barrier after every node
    // phase bounds it).  Fixed nodes' copies are written to both banks at setup.
    const int hbase = 24 * (TS + 2);
    const int bank_stride = local_handoff ? CP.halo_stride : 0;
    auto xat = [&](int off, int bank) {  // x record: own slot, or halo copy in `bank`
      return sm_at<double>(X, off + (off >= hbase ? bank * bank_stride : 0));
    };
    const double scale = P.density_scale / E.max_lump;  // setup_mass relax.cpp:35-43
    const int F0 = Q.f0, NSLOT = Q.node_slots;
    if (e != cur_entry) {
      cur_entry = e;
      s_uni = P.ea_scale * E.ea0;
      for (int i = tid; i < Q.max_pairs * TS; i += T) cent[i] = Q.csr_pairs[i];
      for (int i = tid; i < Q.max_push * TS; i += T) pushd[i] = Q.push_dst[i];
      for (int i = tid; i < TS; i += T) spart[i] = 0.0;
      if (tid < 6) sm_at<double>(X, 24 * TS)[tid] = (tid == 3) ? 1.0 : 0.0;
      if (tid < 3) sm_at<double>(G, 24 * (Q.n_records - 1))[tid] = 0.0;
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = j * T + tid;
        fab[j] = Q.fib_ab[f];
        fgh[j] = Q.fib_gh[f];
        fl0[j] = Q.fib_l0[f];
        // (NaN outside [2^-1000, 2^1000]: the fast-path range test then takes the built-in
        //  operators, fastmath.cuh fiber_fast_ok)
        frl0[j] = (fl0[j] >= 0x1p-1000 && fl0[j] <= 0x1p1000)
                      ? rcp_refined(fl0[j]) : __longlong_as_double(0x7ff8000000000000ll);
        if (!UEA) fs[j] = P.ea_scale * Q.fib_ea[f];
      }
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        npair[j] = Q.csr_npairs[sl];
        npush[j] = Q.push_n[sl];
        nref[j][0] = Q.slot_ref[3 * sl];
        nref[j][1] = Q.slot_ref[3 * sl + 1];
        nref[j][2] = Q.slot_ref[3 * sl + 2];
      }
    }
    auto push_x = [&](int j, int sl, double x0, double x1, double x2, int bank) {
      for (int h = 0; h < npush[j]; ++h) {
        const int d = pushd[h * TS + sl];
        const unsigned a = cl_map(X_sh + (d & 0xffff) + bank * bank_stride,
                                  static_cast<unsigned>(d) >> 16);
        cl_st_f64(a, x0);
        cl_st_f64(a + 8, x1);
        cl_st_f64(a + 16, x2);
      }
    };

    // ---- per-solve setup (relax.cpp:95-145) ----
    double Fm[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fm[i] = P.solve_F[9 * s + i];
    const long long off = P.offsets[p];
    const bool is_base = q < 0;
    double lmin = INFINITY;
#pragma unroll
    for (int j = 0; j < FPT; ++j) {  // reduced_mass_l0 relax.cpp:46-55
      // dummies read the unit segment at TS (in mirror mode a real tail may be a halo node)
      const int ta = (fab[j] & 0xffff) / 24;
      if (ta != TS) {
        const double ma = Q.fib_lt[j * T + tid] * scale;
        const double mb = Q.fib_lh[j * T + tid] * scale;
        fmred[j] = ma * mb / (ma + mb) * fl0[j];
      } else {
        fmred[j] = INFINITY;  // dummy fiber
      }
      if (LAW == 0) {
        const double kt = smax(fabs(law_tangent<0>(SJ(j), 1.0, 0, B)), SJ(j));
        lmin = smin(lmin, fmred[j] / kt);
      }
    }
    double u[NPT][3], vh[NPT][3];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int sl = j * T + tid;
      const int pn = Q.slot_pn[sl];
      const double m = Q.slot_lump[sl] * scale;
      ninv[j] = 1.0 / m;
      ncm[j] = P.damping * m;
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
        const double X0 = nref[j][0], X1 = nref[j][1], X2 = nref[j][2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double fx = Fm[3 * c] * X0 + Fm[3 * c + 1] * X1 + Fm[3 * c + 2] * X2;
          u[j][c] = fx - nref[j][c];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) vh[j][c] = 0.0;
      double* xr = sm_at<double>(X, 24 * sl);
      xr[0] = nref[j][0] + u[j][0];
      xr[1] = nref[j][1] + u[j][1];
      xr[2] = nref[j][2] + u[j][2];
      push_x(j, sl, xr[0], xr[1], xr[2], 0);
      if (sl >= F0 && bank_stride) push_x(j, sl, xr[0], xr[1], xr[2], 1);  // never updated
      if (sl < F0) {
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
      ctl.collapse[0] = ctl.collapse[1] = 0;
      ctl.skip = -1;
    }
    if (LAW == 0) push_wmin(warp_min(lmin));
    const bool det_ok = det3(Fm) > 0;
    cl_sync();  // halo x, CFL minima, control block resets
    double dt_const = 0;
    if (LAW == 0) dt_const = P.dt_safety * sqrt(slots_min(ctl.wmin, C * NW, lane));
    cl_sync();  // wmin consumed before the first fiber phase overwrites it

    int k = 0;
    int target = -1;
    // first pass at which a fiber collapsed (the reference throws there, network.cpp:291):
    // decisive once the lagged verdicts of every earlier pass have been taken
    int cpass = -1;
    double dt_k = 0;
    int status = det_ok ? FIBRA_OK : FIBRA_E_KINEMATICS;
    int conv = 0;

    while (status == FIBRA_OK) {
      // ================= fiber phase (force pass k) =================
      if (warp == NW - 1) {  // reducer warp: owns no fibers
        if (LAW != 0) push_wmin(INFINITY);
        if (target < 0 && k >= 1) {
          // partials of pass k-1 -> every CTA.  Lane l sums slots l, l+32, ... (row i of 32
          // slots is free iff i < F0/32) in four chains, then a butterfly: a short dependency
          // chain (any summation order will do for the speculation)
          constexpr int R = TS / 32;
          const int R0 = F0 >> 5;
          double vf[4] = {0.0, 0.0, 0.0, 0.0}, vx[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < R; ++i) {  // four independent chains of R/4 adds
            const double v = spart[32 * i + lane];
            if (i < R0) vf[i & 3] += v;
            else vx[i & 3] += v;
          }
          double sf = (vf[0] + vf[1]) + (vf[2] + vf[3]), sfix = (vx[0] + vx[1]) + (vx[2] + vx[3]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            sf += __shfl_xor_sync(0xffffffffu, sf, o);
            sfix += __shfl_xor_sync(0xffffffffu, sfix, o);
          }
          if (lane < static_cast<int>(C)) {
            const unsigned a = cl_map(ctl_sh + off_part + ((k - 1) & 1) * 256 + rank * 16, lane);
            cl_st_f64(a, sf);
            cl_st_f64(a + 8, sfix);
          }
          if (k >= 2) {  // verdict for pass k-2 from every CTA's partials (every CTA alike)
            double tf = lane < static_cast<int>(C) ? ctl.part[(k - 2) & 1][lane][0] : 0.0;
            double tx = lane < static_cast<int>(C) ? ctl.part[(k - 2) & 1][lane][1] : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {  // C <= 16
              tf += __shfl_xor_sync(0xffffffffu, tf, o);
              tx += __shfl_xor_sync(0xffffffffu, tx, o);
            }
            // squared form of res <= tol * max(sqrt(tx), floor); a near tie (within ~2e-10
            // in squares) or a tiny threshold is decided exactly with the reference's sums
            const double fl = ctl.force_floor;
            const double e2 = (P.tolerance * P.tolerance) * smax(tx, fl * fl);
            int d = (tf <= e2) ? kDecConv : 0;
            if (!isfinite(tf) || !isfinite(e2)) d |= kDecExact | kDecNonfinite;
            else if (fabs(tf - e2) <= 4e-10 * e2 || e2 < 0x1p-900) d |= kDecExact;
            if (lane == 0)
              ctl.dec = (k - 2 > ctl.skip) ? d : 0;  // decided passes are not re-decided
          }
        }
      } else {
        double kmin = INFINITY;
        bool collapsed = false;
        // fibers in blocks of <= 4 so one block's temporaries are live at a time (FPT = 7
        // shapes otherwise spill); each fiber's local record sits at compact slot j*(T-32)+tid
        auto fiber_block = [&](auto j0c, auto j1c) {
          constexpr int J0 = decltype(j0c)::value, J1 = decltype(j1c)::value;
          bool fast = true;
          double dx[J1 - J0], dy[J1 - J0], dz[J1 - J0], g[J1 - J0];
#pragma unroll
          for (int jj = 0; jj < J1 - J0; ++jj) {
            const int j = J0 + jj;
            const double* xa_ = xat(fab[j] & 0xffff, k & 1);
            const double* xb_ = xat(static_cast<int>(static_cast<unsigned>(fab[j]) >> 16), k & 1);
            dx[jj] = xb_[0] - xa_[0];
            dy[jj] = xb_[1] - xa_[1];
            dz[jj] = xb_[2] - xa_[2];
            bool o1, o2 = true, o3 = true;
            const double len = sqrt_fast(dx[jj] * dx[jj] + dy[jj] * dy[jj] + dz[jj] * dz[jj], o1);
            collapsed |= (len <= 1e-8 * fl0[j]);  // network.cpp:291
            if (LAW == 0) {  // one range test for both divisions (fastmath.cuh)
              const double stretch = div_rcp_raw(len, fl0[j], frl0[j]);
              const double n = law_force<0>(SJ(j), stretch, bo, B);
              g[jj] = div_rcp_raw(n, len, rcp_refined(len));
              o2 = fiber_fast_ok(len, stretch, n);
            } else {
              const double stretch = div_fast_rcp(len, fl0[j], frl0[j], o2);
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
              collapsed |= (len <= 1e-8 * fl0[j]);  // exact length (e.g. 0): network.cpp:291
              const double stretch = len / fl0[j];
              g[jj] = law_force<LAW>(SJ(j), stretch, bo, B) / len;
            }
          }
#pragma unroll
          for (int jj = 0; jj < J1 - J0; ++jj) {  // +g*d: the tail gathers it negated
            const int j = J0 + jj;
            const double g0 = g[jj] * dx[jj], g1 = g[jj] * dy[jj], g2 = g[jj] * dz[jj];
            double* gt = sm_at<double>(G, 24 * (j * (T - 32) + tid));
            gt[0] = g0;
            gt[1] = g1;
            gt[2] = g2;
            if (fgh[j] >= 0) {
              const unsigned a = cl_map(G_sh + (fgh[j] & 0xffffff), static_cast<unsigned>(fgh[j]) >> 24);
              cl_st_f64(a, g0);
              cl_st_f64(a + 8, g1);
              cl_st_f64(a + 16, g2);
            }
          }
        };
        constexpr int B1 = FPT < 4 ? FPT : (FPT + 1) / 2;
        fiber_block(std::integral_constant<int, 0>(), std::integral_constant<int, B1>());
        if constexpr (B1 < FPT)
          fiber_block(std::integral_constant<int, B1>(), std::integral_constant<int, FPT>());
        if (collapsed)
          for (unsigned r = 0; r < C; ++r) cl_st_s32(cl_map(ctl_sh + off_collapse + 4 * (k & 1), r), 1);
        if (LAW != 0) push_wmin(warp_min(kmin));
      }
      if (local_handoff) __syncthreads(); else cl_sync();

      // ================= node phase (pass k) =================
      if (target < 0 && k >= 2 && (cpass < 0 || k - 2 < cpass)) {
        const int d = ctl.dec;
        if ((d & (kDecConv | kDecExact)) || k - 2 == P.max_iterations) {
          target = k - 2;  // replay from the newest checkpoint at or before it
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
              double* xr = sm_at<double>(X, 24 * sl);
              xr[0] = nref[j][0] + u[j][0];
              xr[1] = nref[j][1] + u[j][1];
              xr[2] = nref[j][2] + u[j][2];
              push_x(j, sl, xr[0], xr[1], xr[2], k & 1);
            }
          }
          if (tid == 0) ctl.t = ctl.ck_t[b];
          cpass = -1;
          // discard collapse flags of the passes after the target: once every push of this
          // pass has landed (first barrier), and before anyone pushes again (second)
          cl_sync();
          if (tid == 0) ctl.collapse[0] = ctl.collapse[1] = 0;
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
      // collapse flags of this pass (cluster barrier after the fiber phase), or of the
      // previous pass (local handoff: the last cluster barrier ended node phase k-1)
      // (a replay target always precedes a known collapse, so replays never see one)
      if (cpass < 0 && (local_handoff ? (k >= 1 && ctl.collapse[(k - 1) & 1]) : ctl.collapse[k & 1]))
        cpass = local_handoff ? k - 1 : k;
      if (cpass >= 0 && k - 2 >= cpass - 1) {  // the verdicts of all earlier passes are taken
        status = FIBRA_E_COLLAPSE;
        break;
      }
      const double h_k = 0.5 * dt_k;
      double fk[NPT][3];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        double f0 = 0.0, f1 = 0.0, f2 = 0.0;  // CSR gather, ascending fiber id
        // the next step's pair is loaded one step ahead (predicated: no padding row in the
        // tight config-4 shapes), and the tail's negation is a signed DFMA (dr_kernel.cuh)
        int2 ep = npair[j] > 0 ? cent[sl] : make_int2(0, 0);
#pragma unroll 1
        for (int kp = 0; kp < npair[j]; ++kp) {
          const int2 en = kp + 1 < npair[j] ? cent[(kp + 1) * TS + sl] : ep;
          const double* g0 = sm_at<double>(G, ep.x & 0x7fffffff);
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
          ep = en;
        }
        fk[j][0] = f0;
        fk[j][1] = f1;
        fk[j][2] = f2;
        spart[sl] = f0 * f0 + f1 * f1 + f2 * f2;
      }
      if (k == target) {
        // ---- exact verdict at the target pass: f to the cluster scratch, packed order ----
        const int NFN = E.n_free_nodes, NFIX = E.n_fix_nodes;
        double* SF = scr;
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
          const int pn = Q.slot_pn[j * T + tid];
          if (pn >= 0)
#pragma unroll
            for (int c = 0; c < 3; ++c) SF[3 * pn + c] = fk[j][c];
        }
        __threadfence();
        cl_sync();
        if (warp < 8) {  // norm2_sq partials (4 free, 4 fixed), one warp per chain
          const int r = warp & 3, base = warp < 4 ? 0 : 3 * NFN;
          const int len = warp < 4 ? 3 * NFN : 3 * NFIX;
          const double acc = fold_chain<true>(SF + base, r, 4, len > r ? (len - r + 3) / 4 : 0, lane);
          if (lane == 0) ctl.ex[warp] = acc;
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
          // final state of iteration k -> cluster scratch and (base) PackedStates
          double* SX = scr + 3 * E.n_nodes;
          double* SW = SX + 3 * E.n_nodes;
          const long long soff = P.offsets[ctl.point];
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int sl = j * T + tid;
            const int pn = Q.slot_pn[sl];
            if (pn < 0) continue;
            const double m = Q.slot_lump[sl] * scale;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double fd = 0.0, acc = 0.0, vv = 0.0;
              if (sl < F0 && k >= 1) {
                fd = ncm[j] * vh[j][c];                // kernels_scalar.cpp:15-17
                acc = -(fk[j][c] + fd) * ninv[j];
                vv = vh[j][c] + h_k * acc;             // relax.cpp:166
              }
              SX[3 * pn + c] = nref[j][c] + u[j][c];
              if (sl < F0) SW[3 * pn + c] = m * (vv * vv);
              if (is_base) {
                const long long dd = soff + 3 * pn + c;
                P.u[dd] = u[j][c];
                P.v[dd] = vv;
                P.a[dd] = acc;
                P.f_int[dd] = fk[j][c];
                P.f_damp[dd] = fd;
                P.mass[dd] = m;
                P.inv_mass[dd] = ninv[j];
              }
            }
          }
          break;
        }
        if (tid == 0) ctl.skip = target;  // near tie that did not stop: continue normally
        target = -1;
      }
      // ---- damped update + speculative half step / drift of iteration k+1 ----
      double dt_next;
      if (LAW == 0) {
        dt_next = dt_const;
      } else {
        dt_next = P.dt_safety * sqrt(slots_min(ctl.wmin, C * NW, lane));
      }
      const double h_n = 0.5 * dt_next;
      const bool save = target < 0 && ((k + 1) % kCkInterval == 0);
      const int sb = ((k + 1) / kCkInterval) & 1;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        if (sl < F0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double fd = ncm[j] * vh[j][c];              // kernels_scalar.cpp:15-17
            const double acc = -(fk[j][c] + fd) * ninv[j];
            const double vv = (k >= 1) ? vh[j][c] + h_k * acc : vh[j][c];  // relax.cpp:166
            vh[j][c] = vv + h_n * acc;                          // relax.cpp:155
            u[j][c] = u[j][c] + dt_next * vh[j][c];             // relax.cpp:156
          }
          double* xr = sm_at<double>(X, 24 * sl);
          xr[0] = nref[j][0] + u[j][0];
          xr[1] = nref[j][1] + u[j][1];
          xr[2] = nref[j][2] + u[j][2];
          push_x(j, sl, xr[0], xr[1], xr[2], (k + 1) & 1);
          if (save) {
            double* ck = ckpt + sb * 6 * P.ck_stride;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              ck[c * P.ck_stride + sl] = u[j][c];
              ck[(3 + c) * P.ck_stride + sl] = vh[j][c];
            }
          }
        }
      }
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
    double* SF = scr;
    double* SX = SF + 3 * N;
    double* SW = SX + 3 * N;
    double* SE = SW + 3 * NFN;
    if (status == FIBRA_OK && !zero_iter) {
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const int f = Q.fib_id[j * T + tid];
        if (f >= 0) {  // strain_energy relax.cpp:57-72, from the final x records
          const double* xa_ = xat(fab[j] & 0xffff, k & 1);
          const double* xb_ = xat(static_cast<int>(static_cast<unsigned>(fab[j]) >> 16), k & 1);
          const double dx = xb_[0] - xa_[0];
          const double dy = xb_[1] - xa_[1];
          const double dz = xb_[2] - xa_[2];
          const double len = sqrt(dx * dx + dy * dy + dz * dz);
          SE[f] = law_energy<LAW>(SJ(j), len / fl0[j], fl0[j], bo, B);
        }
      }
    }
    __threadfence();
    cl_sync();
    if (rank == 0) {
      if (status == FIBRA_OK) {  // reference-order reductions (4 partials), one warp each
        if (warp < 12) {
          const int r = warp & 3, which = warp >> 2;
          const double* src = which == 0 ? SF : (which == 1 ? SF + 3 * NFN : SW);
          const int len = which == 1 ? 3 * NFIX : 3 * NFN;
          const int cnt = len > r ? (len - r + 3) / 4 : 0;
          const double acc = which < 2 ? fold_chain<true>(src, r, 4, cnt, lane)
                                       : fold_chain<false>(src, r, 4, cnt, lane);
          if (lane == 0) ctl.ex[warp] = acc;
        }
        if (warp == NW - 1 && !zero_iter) {  // strain_energy: one chain over the fibers
          const double se = fold_chain<false>(SE, 0, 1, M, lane);
          if (lane == 0) ctl.se = se;
        }
        if (warp == NW - 2 && conv) {  // homogenized_stress moments, boundary nodes ascending
          double sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
          for (int c0 = NFN; c0 < N; c0 += 32) {
            const int pn = c0 + lane;
            double rr[3] = {0, 0, 0}, xx[3] = {0, 0, 0};
            if (pn < N)
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                rr[c] = __ldcg(SF + 3 * pn + c);
                xx[c] = __ldcg(SX + 3 * pn + c);
              }
            double pr[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) pr[i] = rr[i / 3] * xx[i % 3];
            const int n = min(32, N - c0);
            for (int s2 = 0; s2 < n; ++s2)
#pragma unroll
              for (int i = 0; i < 9; ++i) sm[i] = sm[i] + __shfl_sync(0xffffffffu, pr[i], s2);
          }
          if (lane == 0)
            for (int i = 0; i < 9; ++i) ctl.mom[i] = sm[i];
        }
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
            const double se = ctl.se;
            o.kinetic_fraction = (ke + se) > 0 ? ke / (ke + se) : 0.0;
          }
          if (conv) {  // homogenized_stress moment sums, boundary nodes ascending
            for (int i = 0; i < 9; ++i) o.moment[i] = ctl.mom[i];
            o.box_volume = E.box_volume;
          } else {
            o.status = is_base ? FIBRA_E_NOT_CONVERGED : FIBRA_E_PROBE_FAILED;
          }
        }
        P.out[s] = o;
        trace_end(P, s, n_done);
        if (is_base) {
          P.t[p] = ctl.t;
          if (status == FIBRA_OK) {
            P.iters[p] += n_done;
            P.converged[p] = static_cast<unsigned char>(conv);
          } else {
            P.converged[p] = 0;
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
    }
    if (is_base) {  // every CTA wrote part of the base state its probes warm-start from
      __threadfence();
      cl_sync();
      if (rank == 0 && tid == 0) publish_base(P, p, P.out[s].status == FIBRA_OK ? 1 : 2);
    }
    cl_sync();
  }
#undef SJ
}

}  // namespace fibra_b200
