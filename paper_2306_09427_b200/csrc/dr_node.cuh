// Node-centric persistent dynamic-relaxation kernel: one CTA solves one RVE at a time,
// pulling (point, solve) tickets from the same device queue as dr_kernel.cuh, with ONE
// barrier per DR iteration (linear law).
//
// Reference path this replaces (paths under /root/reference/proj):
//   relax_solve           src/relax.cpp:93-191   (setup :95-145, hot loop :148-179)
//   internal_forces_cfl   src/network.cpp:275-324 (force law :16-53)
//   L1 kernels            src/kernels_scalar.cpp:7-65
//   apply_affine_bc       src/network.cpp:254-269
//   homogenized_stress    src/network.cpp:341-372 (moment sums; finished in post_kernel)
//
// Design.  Each thread owns NPT node slots (u and the half-step velocity in registers).
// Per pass it walks its node's incident fibers in ascending reference fiber id -- the
// accumulation order of network.cpp:298-303 -- evaluates each fiber itself and subtracts
// g*d' from a force that starts at +0.0, where d' = x_other - x_own:
//   tail node: d' = x_head - x_tail = d, reference f_tail -= g*d                 -> same;
//   head node: d' = x_tail - x_head = -d exactly (round-to-nearest is odd), so
//              g*d' = -(g*d) and f - g*d' = f + g*d, the reference's f_head += g*d.
// Length, stretch and g depend on d only through squares and are bitwise identical at
// both ends.  Every fiber is therefore evaluated twice (once per end), but the fiber ->
// node hand-off through shared memory and its barrier disappear: x is double-buffered by
// pass parity, so the only barrier of an iteration separates the x writes of pass k+1
// from the x reads of pass k.  (The nonlinear law adds one barrier: dt of iteration k+1
// is the CFL minimum over all fibers of pass k.)
//
// Incidences are stored step-major per warp (row r, lane l at 32 r + l: consecutive lanes,
// consecutive words) in shared memory: the other node's x-record byte offset and the pair
// (l0, rcp_refined(l0)).  Nodes are degree-sorted into warps (host/node_schedule.cpp), a
// warp walks max(degree) steps, and the x-record placement spreads each gather step over
// the 16 bank pairs.
//
// Convergence off the critical path (as dr_kernel.cuh): every warp adds its nodes' |f|^2
// (free or fixed) into a per-pass shared slot; the next pass reads the approximate verdict
// (|R - eps| <= 1e-10 eps, or non-finite, goes through the exact reference-order decision);
// a stop at k restores the newest checkpoint <= k, replays (bit-identical) and decides at k
// with the reference's 4-lane sums (kernels_scalar.cpp:20-33).
#pragma once

#include <cstdint>

#include "dr_kernel.cuh"
#include "fastmath.cuh"
#include "fibra_cuda.h"
#include "tensor.cuh"

namespace fibra_b200 {

struct NodeEntryDev {      // one RveLibrary entry for dr_node_kernel, in slot order
  int n_nodes, n_fibers, n_free_nodes, n_fix_nodes;
  int f0, node_slots, n_rows, pad0;  // n_rows: incidence rows (sum over warps of max degree)
  double max_lump, max_ea, box_volume, pad1;
  const int* slot_pn;      // [node_slots] packed node id, -1 empty
  const double* slot_ref;  // [3*node_slots] reference coordinates
  const double* slot_lump; // [node_slots] lumping weight (1 when empty)
  const int* slot_deg;     // [node_slots] incident fibers
  const int* group_row0;   // [node_slots/32 + 1] first incidence row of each warp group
  const int* inc_x;        // [32*n_rows] x byte offset of the other end (step-major)
  const double* inc_l0;    // [32*n_rows] rest length
  const double* inc_ea;    // [32*n_rows] area*modulus
  const double* inc_lump;  // [32*n_rows] lumping weight of the other end (CFL reduced mass)
  const int* fib_a;        // [n_fibers] packed node of the tail (exit strain energy)
  const int* fib_b;        // [n_fibers] packed node of the head
  const double* fib_l0;    // [n_fibers]
  const double* fib_ea;    // [n_fibers]
};

struct __align__(16) NodeCtl {
  int solve, point, q, entry;
  int flag, dec, skip, pad;
  double sum[3][2];        // per pass mod 3: sum |f|^2 over free / fixed nodes (approximate)
  int coll[3];             // per pass mod 3: a fiber collapsed
  int pad2;
  double ck_t[2], ck_dt[2];
  double warp_min[2][32];
  double ex[12];
  double t;
  double force_floor;
};

template <int T, int NPT, int LAWBO, int MINB, bool UEA>
__global__ void __launch_bounds__(T, MINB) dr_node_kernel(DrParams P) {
  constexpr int LAW = LAWBO & 1;
  constexpr int bo = LAWBO >> 1;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ NodeCtl ctl;
  constexpr int NW = T / 32;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // shared layout: [XB0 | XB1] x records by pass parity (P.x_bytes each)
  //                [IX: int inc_x][IL: double2 (l0, rcp l0)][IE: double ea][IM: double mred]
  // (the incidence arrays have P.csr_cap entries; exit scratch reuses everything)
  unsigned char* XB = smem;
  const int cap = P.csr_cap;
  int* IX = reinterpret_cast<int*>(smem + 2 * P.x_bytes);
  double2* IL = reinterpret_cast<double2*>(smem + 2 * P.x_bytes + ((4 * cap + 15) & ~15));
  double* IE = reinterpret_cast<double*>(IL + cap);
  double* IM = IE + (UEA ? 0 : cap);
  double* ckpt = P.ckpt + static_cast<size_t>(blockIdx.x) * 12 * P.ck_stride;
  const double B = P.nonlinearity;

  int cur_entry = -1;
  bool first_ticket = true;
  double s_uni = 0;
  int deg[NPT], row0[NPT], nsteps[NPT];
#define NREF(j, c) __ldg(E.slot_ref + 3 * ((j) * T + tid) + (c))

  for (;;) {
    if (tid == 0) {  // ticket: same queue protocol as dr_persistent_kernel
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
        ctl.flag = flag;
        trace_start(P, s);
      }
      ctl.solve = s;
    }
    __syncthreads();
    const int s = ctl.solve;
    if (s < 0) break;
    const int p = ctl.point, q = ctl.q, e = ctl.entry;
    if (!ctl.flag) {
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

    const NodeEntryDev& E = P.nentries[e];
    const double scale = P.density_scale / E.max_lump;  // setup_mass relax.cpp:35-43
    const int F0 = E.f0;
    if (e != cur_entry) {  // incidence tables into shared memory (exit scratch clobbers them)
      cur_entry = e;
      s_uni = P.ea_scale * E.fib_ea[0];
      const int ninc = 32 * E.n_rows;
      for (int i = tid; i < ninc; i += T) {
        IX[i] = E.inc_x[i];
        const double l0 = E.inc_l0[i];
        IL[i] = make_double2(l0, rcp_refined(l0));
        if (!UEA) IE[i] = P.ea_scale * E.inc_ea[i];
      }
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        deg[j] = E.slot_deg[sl];
        row0[j] = E.group_row0[sl >> 5];
        nsteps[j] = E.group_row0[(sl >> 5) + 1] - row0[j];
      }
    }
    // ---- per-solve setup (relax.cpp:95-145) ----
    double Fm[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fm[i] = P.solve_F[9 * s + i];
    const long long off = P.offsets[p];
    const bool is_base = q < 0;
    double u[NPT][3], vh[NPT][3], ninv[NPT], ncm[NPT];
    double lmin = INFINITY;
    unsigned char* X0 = XB;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int sl = j * T + tid;
      const int pn = E.slot_pn[sl];
      const double lump = E.slot_lump[sl];
      const double m = lump * scale;
      ninv[j] = 1.0 / m;
      ncm[j] = P.damping * m;
      // reduced_mass_l0 (relax.cpp:46-55) of every incident fibre, (ma*mb)/(ma+mb)*l0 with
      // a = tail, b = head; the product and the sum are symmetric, so the order is free
      for (int st = 0; st < deg[j]; ++st) {
        const int ix = 32 * (row0[j] + st) + (sl & 31);
        const double mb = E.inc_lump[ix] * scale;
        const double mred = m * mb / (m + mb) * E.inc_l0[ix];
        if (LAW == 0) {
          const double sj = UEA ? s_uni : P.ea_scale * E.inc_ea[ix];
          const double kt = smax(fabs(law_tangent<0>(sj, 1.0, 0, B)), sj);
          lmin = smin(lmin, mred / kt);
        } else {
          IM[ix] = mred;
        }
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
      double* xr = sm_at<double>(X0, 24 * sl);
      xr[0] = NREF(j, 0) + u[j][0];
      xr[1] = NREF(j, 1) + u[j][1];
      xr[2] = NREF(j, 2) + u[j][2];
      if (sl >= F0) {  // fixed nodes never move: both buffers
        double* xr1 = sm_at<double>(X0 + P.x_bytes, 24 * sl);
        xr1[0] = xr[0];
        xr1[1] = xr[1];
        xr1[2] = xr[2];
      } else {  // checkpoint "resume at pass 0": u_0, v = 0
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
      for (int i = 0; i < 3; ++i) {
        ctl.sum[i][0] = ctl.sum[i][1] = 0.0;
        ctl.coll[i] = 0;
      }
    }
    if (LAW == 0) {
      lmin = warp_min(lmin);
      if (lane == 0) ctl.warp_min[0][warp] = lmin;
    }
    const bool det_ok = det3(Fm) > 0;
    __syncthreads();
    double dt_const = 0;
    if (LAW == 0) {
      double mn = INFINITY;
      for (int w = 0; w < NW; ++w) mn = smin(mn, ctl.warp_min[0][w]);
      dt_const = P.dt_safety * sqrt(mn);
    }

    int k = 0;              // force pass this iteration evaluates
    int target = -1;        // pass at which to stop and decide exactly (replay mode)
    double dt_k = 0;        // dt of iteration k (0 for the initial pass)
    int status = det_ok ? FIBRA_OK : FIBRA_E_KINEMATICS;
    int conv = 0;
    bool rewrite_fixed = false;
    double fk[NPT][3];

    while (status == FIBRA_OK) {
      // ---- verdict of pass k-1 (written before the last barrier) ----
      if (target < 0 && k >= 1) {
        const int sp = (k - 1) % 3;
        if (ctl.coll[sp]) {  // network.cpp:291 throws inside the force pass of k-1
          status = FIBRA_E_COLLAPSE;
          k -= 1;            // the collapsed pass (committed, then threw)
          break;
        }
        const double sf = ctl.sum[sp][0], sfix = ctl.sum[sp][1];
        const double res = sqrt(sf);
        const double eps = P.tolerance * smax(sqrt(sfix), ctl.force_floor);
        int d = (res <= eps) ? kDecConv : 0;
        if (!isfinite(res) || !isfinite(eps)) d |= kDecExact | kDecNonfinite;
        else if (fabs(res - eps) <= 1e-10 * eps) d |= kDecExact;
        if (k - 1 <= ctl.skip) d = 0;  // decided exactly already ("continue" at a near tie)
        if ((d & (kDecConv | kDecExact)) || k - 1 == P.max_iterations) {
          target = k - 1;
          k = target / kCkInterval * kCkInterval;  // newest checkpoint <= target
          const int b = (k / kCkInterval) & 1;
          dt_k = ctl.ck_dt[b];
          const double* ck = ckpt + b * 6 * P.ck_stride;
          unsigned char* Xk = XB + (k & 1) * P.x_bytes;
#pragma unroll
          for (int j = 0; j < NPT; ++j) {
            const int sl = j * T + tid;
            if (sl < F0) {
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                u[j][c] = __ldcg(ck + c * P.ck_stride + sl);
                vh[j][c] = __ldcg(ck + (3 + c) * P.ck_stride + sl);
              }
              double* xr = sm_at<double>(Xk, 24 * sl);
              xr[0] = NREF(j, 0) + u[j][0];
              xr[1] = NREF(j, 1) + u[j][1];
              xr[2] = NREF(j, 2) + u[j][2];
            }
          }
          __syncthreads();  // everyone has read ctl.* of pass k-1 before it is reset
          if (tid == 0) {
            ctl.t = ctl.ck_t[b];
            for (int i = 0; i < 3; ++i) {
              ctl.sum[i][0] = ctl.sum[i][1] = 0.0;
              ctl.coll[i] = 0;
            }
          }
          rewrite_fixed = false;
          __syncthreads();
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
      if (tid == 0) {  // the slot of pass k+1 (read for the last time in pass k-1)
        const int sn = (k + 1) % 3;
        ctl.sum[sn][0] = ctl.sum[sn][1] = 0.0;
        ctl.coll[sn] = 0;
      }

      // ================= forces of pass k =================
      const unsigned char* Xc = XB + (k & 1) * P.x_bytes;
      bool collapsed = false;
      double kmin = INFINITY;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        const double x0 = NREF(j, 0) + u[j][0];
        const double x1 = NREF(j, 1) + u[j][1];
        const double x2 = NREF(j, 2) + u[j][2];
        double f0 = 0.0, f1 = 0.0, f2 = 0.0;
        const int n_j = deg[j], ns = nsteps[j];
        // one incidence, fast path only: every lane of the warp evaluates its row (lanes past
        // their degree read the padding entry, x of slot 0 and l0 = 1, and discard it)
        struct Inc {
          double dx, dy, dz, len, g, l0;
          bool ok;
        };
        auto eval = [&](int st) {
          Inc r;
          const int ix = 32 * (row0[j] + st) + lane;
          const double* xo = sm_at<const double>(const_cast<unsigned char*>(Xc), IX[ix]);
          const double2 lr = IL[ix];
          r.dx = xo[0] - x0;  // d' = x_other - x_own
          r.dy = xo[1] - x1;
          r.dz = xo[2] - x2;
          r.l0 = lr.x;
          const double sj = UEA ? s_uni : IE[ix];
          bool o1, o2, o3 = true;
          r.len = sqrt_fast(r.dx * r.dx + r.dy * r.dy + r.dz * r.dz, o1);
          const double stretch = div_fast_rcp_i(r.len, lr.x, lr.y, o2);
          if (LAW == 0) {
            r.g = div_fast_i(law_force<0>(sj, stretch, bo, B), r.len, o3);
          } else {
            r.g = law_force<LAW>(sj, stretch, bo, B) / r.len;
            const double kt = smax(fabs(law_tangent<LAW>(sj, stretch, bo, B)), sj);
            if (st < n_j) kmin = smin(kmin, IM[ix] / kt);
          }
          r.ok = (o1 && o2 && o3) || st >= n_j;
          return r;
        };
        auto slow = [&](Inc& r, int st) {  // rare: special operands -> built-in ops
          if (!r.ok) {
            const double sj = UEA ? s_uni : IE[32 * (row0[j] + st) + lane];
            r.len = sqrt(r.dx * r.dx + r.dy * r.dy + r.dz * r.dz);
            r.g = law_force<LAW>(sj, r.len / r.l0, bo, B) / r.len;
          }
        };
        auto add = [&](const Inc& r, int st) {  // f_tail -= g*d; f_head += g*d (network.cpp:298-303)
          if (st < n_j) {
            collapsed |= le_nonneg_bits(r.len, 1e-8 * r.l0);  // len <= 1e-8 l0, network.cpp:291
            f0 = f0 - r.g * r.dx;
            f1 = f1 - r.g * r.dy;
            f2 = f2 - r.g * r.dz;
          }
        };
        int st = 0;
        for (; st + 1 < ns; st += 2) {  // two incidences in flight, accumulated in order
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
        // approximate |f|^2 of the warp group (free or fixed), tree order
        const double part = warp_sum(f0 * f0 + f1 * f1 + f2 * f2);
        if (lane == 0) atomicAdd(&ctl.sum[k % 3][sl < F0 ? 0 : 1], part);
      }
      if (collapsed) ctl.coll[k % 3] = 1;
      if (LAW != 0) {
        kmin = warp_min(kmin);
        if (lane == 0) ctl.warp_min[k & 1][warp] = kmin;
        __syncthreads();  // dt of iteration k+1 = CFL minimum over all fibres of pass k
      }

      const double h_k = 0.5 * dt_k;
      if (k == target) {
        // ---- exact verdict at the target pass (reference-order norms) ----
        double* SF = reinterpret_cast<double*>(XB + ((k + 1) & 1) * P.x_bytes);
        __syncthreads();  // (the buffer of pass k+1 is free: pass k-1 reads are done)
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
          // final state of iteration k into the exit scratch (SF holds f) and, for base
          // solves, into the PackedStates (batch.cpp:169-176)
          double* SX = reinterpret_cast<double*>(IX);
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
        for (int w = 0; w < NW; ++w) mn = smin(mn, ctl.warp_min[k & 1][w]);
        dt_next = P.dt_safety * sqrt(mn);
      }
      const double h_n = 0.5 * dt_next;
      const bool save = target < 0 && ((k + 1) % kCkInterval == 0);
      const int sb = ((k + 1) / kCkInterval) & 1;
      unsigned char* Xn = XB + ((k + 1) & 1) * P.x_bytes;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int sl = j * T + tid;
        double* xr = sm_at<double>(Xn, 24 * sl);
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
      __syncthreads();
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
    __syncthreads();
    const double* SF = reinterpret_cast<const double*>(XB + ((k + 1) & 1) * P.x_bytes);
    double* SX = reinterpret_cast<double*>(IX);                // x = ref + u (3N)
    double* SW = SX + 3 * N;                                   // m v^2, free dofs (3*NFN)
    double* SE = SW + 3 * NFN;                                 // strain energy per fiber (M)
    if (status == FIBRA_OK && !zero_iter) {
      for (int f = tid; f < M; f += T) {  // strain_energy relax.cpp:57-72
        const int ta = E.fib_a[f], hb = E.fib_b[f];
        const double dx = SX[3 * hb] - SX[3 * ta];
        const double dy = SX[3 * hb + 1] - SX[3 * ta + 1];
        const double dz = SX[3 * hb + 2] - SX[3 * ta + 2];
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        const double l0 = E.fib_l0[f];
        const double sj = UEA ? s_uni : P.ea_scale * E.fib_ea[f];
        SE[f] = law_energy<LAW>(sj, len / l0, l0, bo, B);
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
    cur_entry = -1;  // the exit scratch overwrote the incidence tables
    if (base_solve) {
      __threadfence();
      __syncthreads();
      if (tid == 0) publish_base(P, p_, P.out[s_].status == FIBRA_OK ? 1 : 2);
    }
    __syncthreads();
  }
#undef NREF
}

}  // namespace fibra_b200
