// B200 batched RVE solver: device context, prep/post kernels and the C-ABI
// (include/fibra_cuda.h).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// --fmad=false -lineinfo (see paper_2306_09427_b200/build.py).
//
// One fibra_cuda_solve == the reference batch_response (proj/src/batch.cpp:155-187) for
// every point, split into three launches on the context stream:
//   prep_kernel   per point: polar_decompose(F) (tensor.cpp:203-224), probe stretches
//                 U + h T_q (stiffness.cpp:86-127); one thread per point
//   dr_persistent_kernel   all DR solves (bases first, then probes) from a ticket queue
//   post_kernel   per point: A from probes (stiffness.cpp:15-41), C = push-forward(A, F)
//                 (tensor.cpp:286-300), sigma = R sigma_U R^T (stiffness.cpp:171-173)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "dr_kernel.cuh"
#include "host/schedule.hpp"
#include "fibra_cuda.h"
#include "tensor.cuh"

namespace fibra_b200 {

static_assert(sizeof(fibra_point_result) == 760, "fibra_point_result ABI layout");

struct PrepOut {
  double R[9];
  double U[6];
  double h;
  int status;
  int pad;
};

__global__ void prep_kernel(int n, const double* __restrict__ F, int want_tangent,
                            double fd_rel_step, PrepOut* prep, double* solve_F, int* solve_skip,
                            int* base_flag, int* done_list, int sched_mode,
                            const double* __restrict__ hint, unsigned long long* key) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double f[9];
  for (int i = 0; i < 9; ++i) f[i] = F[9 * p + i];
  PrepOut o = {};
  base_flag[p] = 0;
  done_list[p] = -1;
  // schedule key (ascending = started first), unique through the point index in the low word
  unsigned hi = 0;
  if (sched_mode == FIBRA_SCHED_STRAIN) {
    double e2 = 0;  // |F^T F - I|^2, fp64 only for ordering
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double c = f[i] * f[j] + f[3 + i] * f[3 + j] + f[6 + i] * f[6 + j] - (i == j);
        e2 += c * c;
      }
    const float k = static_cast<float>(sqrt(e2));
    hi = k == k ? __float_as_uint(k) : 0xffffffffu;
  } else if (sched_mode == FIBRA_SCHED_HINT) {
    const float k = static_cast<float>(hint[p]);
    hi = (k == k && k > 0) ? ~__float_as_uint(k) : 0xffffffffu;
  }
  key[p] = (static_cast<unsigned long long>(hi) << 32) | static_cast<unsigned>(p);
  if (!polar_decompose(f, o.R, o.U)) {  // KinematicsError -> failed point
    o.status = FIBRA_E_KINEMATICS;
    solve_skip[p] = FIBRA_E_KINEMATICS;
    for (int i = 0; i < 9; ++i) solve_F[9 * p + i] = 0.0;
  } else {
    solve_skip[p] = 0;
    sym_full(o.U, solve_F + 9 * p);
  }
  if (want_tangent) {
    o.h = fd_rel_step * sym_frobenius(o.U);  // probe_step stiffness.cpp:125-127
    for (int q = 0; q < 6; ++q) {
      const int s = n + 6 * p + q;
      double dir[6], up[6];
      probing_direction(q, dir);
      for (int i = 0; i < 6; ++i) up[i] = o.U[i] + dir[i] * o.h;
      sym_full(up, solve_F + 9 * s);
      if (o.status) {
        solve_skip[s] = o.status;
      } else {
        solve_skip[s] = det3(solve_F + 9 * s) > 0 ? 0 : FIBRA_E_PROBE_FAILED;  // :95-96
      }
    }
  }
  prep[p] = o;
}

// order[rank of key[p]] = p (keys are unique): a counting rank, O(n^2 / 256) smem compares,
// a few microseconds at thousands of points
__global__ void rank_kernel(int n, const unsigned long long* __restrict__ key, int* order) {
  __shared__ unsigned long long tile[256];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long k = p < n ? key[p] : 0;
  int rank = 0;
  for (int b = 0; b < n; b += 256) {
    __syncthreads();
    if (b + static_cast<int>(threadIdx.x) < n) tile[threadIdx.x] = key[b + threadIdx.x];
    __syncthreads();
    const int m = min(256, n - b);
    for (int j = 0; j < m; ++j) rank += tile[j] < k;
  }
  if (p < n) order[rank] = p;
}

// homogenized_stress (network.cpp:341-372) from the boundary moment sums of a converged
// solve, then pull_back_stress (tensor.cpp:309-315) at the solve's stretch Fs
__device__ bool finish_stress(const SolveOut& o, const double* Fs, double* sigma,
                              double* asym_out, double* pk2) {
  const double vol = det3(Fs) * o.box_volume;
  double raw[9];
  for (int i = 0; i < 9; ++i) raw[i] = o.moment[i] / vol;
  double asym = 0, mag = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      asym += (raw[3 * i + j] - raw[3 * j + i]) * (raw[3 * i + j] - raw[3 * j + i]);
      mag += raw[3 * i + j] * raw[3 * i + j];
    }
  sym_from_full(raw, sigma);
  *asym_out = mag > 0 ? sqrt(asym / mag) : 0.0;
  return pull_back_stress(sigma, Fs, pk2);
}

__global__ void post_kernel(int n, const double* __restrict__ F, int want_tangent,
                            const PrepOut* __restrict__ prep, const SolveOut* __restrict__ out,
                            const double* __restrict__ solve_F, fibra_point_result* res) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  fibra_point_result r;
  memset(&r, 0, sizeof r);
  r.failed_probe = -1;
  const PrepOut& pr = prep[p];
  const SolveOut& b = out[p];
  int status = pr.status ? pr.status : b.status;
  int failed_probe = -1;
  int64_t its = b.iterations;
  double sigma_u[6], asym = 0, pk2[6], probe_pk2[36];
  if (!status && !finish_stress(b, solve_F + 9 * p, sigma_u, &asym, pk2))
    status = FIBRA_E_KINEMATICS;
  if (!status && want_tangent) {
    for (int q = 0; q < 6 && !status; ++q) {
      const int s = n + 6 * p + q;
      const SolveOut& o = out[s];
      double sq[6], aq;
      if (o.status || !finish_stress(o, solve_F + 9 * s, sq, &aq, probe_pk2 + 6 * q)) {
        status = FIBRA_E_PROBE_FAILED;
        failed_probe = q;
      } else {
        its += o.iterations;
      }
    }
    if (!status) {
      if (!material_stiffness_from_probes(pr.U, pk2, probe_pk2, pr.h, r.material_a))
        status = FIBRA_E_SINGULAR;
      else {
        double f[9];
        for (int i = 0; i < 9; ++i) f[i] = F[9 * p + i];
        if (!push_forward_stiffness(r.material_a, f, r.spatial_c)) status = FIBRA_E_KINEMATICS;
      }
    }
  }
  if (status) {  // failed point: value-initialized response (batch.cpp:177-185)
    fibra_point_result z;
    memset(&z, 0, sizeof z);
    z.failed_probe = failed_probe;
    z.status = status;
    res[p] = z;
    return;
  }
  rotate_stress(pr.R, sigma_u, r.sigma);
  for (int i = 0; i < 6; ++i) r.pk2[i] = pk2[i];
  r.stress_asymmetry = asym;
  r.base_report.iterations = b.iterations;
  r.base_report.residual = b.residual;
  r.base_report.eps_eff = b.eps_eff;
  r.base_report.kinetic_fraction = b.kinetic_fraction;
  r.base_report.dt = b.dt;
  r.base_report.converged = b.converged;
  r.base_report.energy_drift = 0;
  r.solves = want_tangent ? 7 : 1;
  r.relax_iterations = its;
  r.failed_probe = -1;
  r.status = FIBRA_OK;
  res[p] = r;
}

// Self-test of fastmath.cuh: div_fast / sqrt_fast (+ the built-in fallback the DR kernel
// applies when the predicate fails) against the built-in IEEE operators, bit for bit.
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

__device__ __forceinline__ double operand(unsigned long long r, int mode) {
  // mode 0: |exponent| <= 64 around 1; mode 1: any finite exponent; mode 2: raw bits
  // (zeros, denormals, inf, NaN); mode 3: short-mantissa values (exact cases)
  const unsigned long long sign = (r >> 63) << 63;
  const unsigned long long mant = r & 0x000fffffffffffffull;
  unsigned long long e;
  if (mode == 0) e = 1023 - 64 + ((r >> 52) & 127);
  else if (mode == 1) e = 1 + ((r >> 52) % 2046);
  else if (mode == 2) return __longlong_as_double(static_cast<long long>(r));
  else return static_cast<double>(static_cast<long long>(r >> 40) % 4096) * 0.125;
  return __longlong_as_double(static_cast<long long>(sign | (e << 52) | mant));
}

__device__ __forceinline__ bool same_bits(double x, double y) {
  return __double_as_longlong(x) == __double_as_longlong(y) || (isnan(x) && isnan(y));
}

__global__ void fastmath_selftest_kernel(unsigned long long n, unsigned long long seed,
                                         unsigned long long* bad) {
  unsigned long long local = 0;
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long r0 = mix64(seed ^ (2 * i)), r1 = mix64(seed ^ (2 * i + 1));
    const int mode = static_cast<int>(i & 3);
    const double a = operand(r0, mode), b = operand(r1, mode == 3 ? 0 : mode);
    bool ok;
    double q = div_fast(a, b, ok);
    if (!ok) q = a / b;
    local += !same_bits(q, a / b);
    const double x = mode == 2 ? a : fabs(a);
    double s = sqrt_fast(x, ok);
    if (!ok) s = sqrt(x);
    local += !same_bits(s, sqrt(x));
  }
  if (local) atomicAdd(bad, local);
}

// FP64 pipe peak probe: 8 independent DADD chains per thread, 1024 threads per SM
__global__ void fp64_peak_kernel(double* sink, int iters, double c) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] + c;
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) sink[threadIdx.x] = s;
}

// ---------------------------------------------------------------------------------
// kernel variants: T threads, FPT fibers and NPT nodes per thread, force law
// ---------------------------------------------------------------------------------
using KernelFn = void (*)(DrParams);

struct Variant {
  int T, FPT, NPT, MINB;
  KernelFn fn[2][2];  // [law: linear, exponential][uniform EA]
};

// Ordered by preference: the first variant whose capacity covers every library entry wins.
// MINB = 2 keeps two CTAs (two RVEs) per SM so one CTA's barrier wait is covered by the
// other's work.
#define FB_V(T, F, N, B)                                                                 \
  {T, F, N, B,                                                                             \
   {{&dr_persistent_kernel<T, F, N, 0, B, false>, &dr_persistent_kernel<T, F, N, 0, B, true>}, \
    {&dr_persistent_kernel<T, F, N, 1, B, false>, &dr_persistent_kernel<T, F, N, 1, B, true>}}}
static const Variant kVariants[] = {
    FB_V(256, 3, 1, 2),  // <= 256 node slots, <= 768 fibers
    FB_V(384, 3, 1, 2),  // <= 384 node slots, <= 1152 fibers (config 1/2 networks)
    FB_V(512, 2, 1, 2),  // <= 512 node slots, <= 1024 fibers
    FB_V(512, 4, 1, 1),  // <= 512 node slots, <= 2048 fibers
    FB_V(512, 6, 2, 1),  // <= 1024 node slots, <= 3072 fibers
    FB_V(768, 7, 2, 1),  // <= 1536 node slots, <= 5376 fibers (ragged config-3 tail)
};
#undef FB_V

struct DeviceEntry {
  EntryDev dev;
  Schedule sched;
  std::vector<void*> allocs;
  bool config_ok = true;
  std::string config_err;
};

}  // namespace fibra_b200

using namespace fibra_b200;

struct fibra_ctx {
  int device = 0;
  int n_sm = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  std::string err;
  std::vector<DeviceEntry> entries;
  EntryDev* d_entries = nullptr;
  const Variant* variant = nullptr;
  bool uniform_ea = false;  // every entry has a single area*modulus over its fibers
  int x_bytes = 0, g_bytes = 0, part_slots = 0, csr_cap = 0, ck_stride = 0;
  // points
  int n_points = 0;
  std::vector<int32_t> entry_of_point;
  std::vector<long long> offsets;
  int* d_entry_of_point = nullptr;
  long long* d_offsets = nullptr;
  double* d_state[8] = {};  // u v a f_int f_damp mass inv_mass t
  long long* d_iters = nullptr;
  unsigned char* d_conv = nullptr;
  int sched_mode = FIBRA_SCHED_STRAIN;
  double* d_hint = nullptr;  // FIBRA_SCHED_HINT costs (n_points)
  // per-call scratch
  int cap_points = 0;
  double* d_F = nullptr;
  double* d_solveF = nullptr;
  int* d_skip = nullptr;
  PrepOut* d_prep = nullptr;
  SolveOut* d_out = nullptr;
  int* d_flag = nullptr;
  int* d_done = nullptr;
  int* d_order = nullptr;
  unsigned long long* d_key = nullptr;
  fibra_point_result* d_res = nullptr;
  double* h_F = nullptr;                 // pinned staging
  fibra_point_result* h_res = nullptr;   // pinned staging
  double* d_ckpt = nullptr;
  size_t ckpt_cap = 0;
  int* d_ticket = nullptr;
  unsigned long long* d_counters = nullptr;
  cudaEvent_t ev[4] = {};
  int last_solves = 0;
  int last_launches = 0;
  unsigned long long* phase_prof = nullptr;
  size_t phase_prof_n = 0;
};

namespace {

int set_err(fibra_ctx* c, int code, const std::string& what) {
  if (c) c->err = what;
  return code;
}

#define FB_CUDA(ctx, call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_err(ctx, FIBRA_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
int dalloc(fibra_ctx* c, T** p, size_t n) {
  if (n == 0) n = 1;
  FB_CUDA(c, cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  return FIBRA_OK;
}

void free_points(fibra_ctx* c) {
  cudaFree(c->d_entry_of_point);
  cudaFree(c->d_offsets);
  for (auto& p : c->d_state) cudaFree(p), p = nullptr;
  cudaFree(c->d_iters);
  cudaFree(c->d_conv);
  cudaFree(c->d_hint);
  c->d_hint = nullptr;
  if (c->sched_mode == FIBRA_SCHED_HINT) c->sched_mode = FIBRA_SCHED_STRAIN;
  c->d_entry_of_point = nullptr;
  c->d_offsets = nullptr;
  c->d_iters = nullptr;
  c->d_conv = nullptr;
  c->n_points = 0;
}

void free_scratch(fibra_ctx* c) {
  cudaFree(c->d_F);
  cudaFree(c->d_solveF);
  cudaFree(c->d_skip);
  cudaFree(c->d_prep);
  cudaFree(c->d_out);
  cudaFree(c->d_flag);
  cudaFree(c->d_done);
  cudaFree(c->d_order);
  cudaFree(c->d_key);
  cudaFree(c->d_res);
  cudaFreeHost(c->h_F);
  cudaFreeHost(c->h_res);
  c->d_F = c->d_solveF = nullptr;
  c->d_skip = c->d_flag = c->d_done = c->d_order = nullptr;
  c->d_key = nullptr;
  c->d_prep = nullptr;
  c->d_out = nullptr;
  c->d_res = nullptr;
  c->h_F = nullptr;
  c->h_res = nullptr;
  c->cap_points = 0;
}

void free_library(fibra_ctx* c) {
  for (auto& e : c->entries)
    for (void* p : e.allocs) cudaFree(p);
  c->entries.clear();
  cudaFree(c->d_entries);
  c->d_entries = nullptr;
  c->variant = nullptr;
}

int ensure_scratch(fibra_ctx* c, int n) {
  if (n <= c->cap_points) return FIBRA_OK;
  free_scratch(c);
  const size_t ns = 7 * static_cast<size_t>(n);
  int rc;
  if ((rc = dalloc(c, &c->d_F, 9 * static_cast<size_t>(n)))) return rc;
  if ((rc = dalloc(c, &c->d_solveF, 9 * ns))) return rc;
  if ((rc = dalloc(c, &c->d_skip, ns))) return rc;
  if ((rc = dalloc(c, &c->d_prep, n))) return rc;
  if ((rc = dalloc(c, &c->d_out, ns))) return rc;
  if ((rc = dalloc(c, &c->d_flag, n))) return rc;
  if ((rc = dalloc(c, &c->d_done, n))) return rc;
  if ((rc = dalloc(c, &c->d_order, n))) return rc;
  if ((rc = dalloc(c, &c->d_key, n))) return rc;
  if ((rc = dalloc(c, &c->d_res, n))) return rc;
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_F), 9 * sizeof(double) * n));
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_res), sizeof(fibra_point_result) * n));
  c->cap_points = n;
  return FIBRA_OK;
}

size_t align16(size_t b) { return (b + 15) & ~static_cast<size_t>(15); }

size_t smem_bytes(const fibra_ctx* c) {
  return static_cast<size_t>(c->x_bytes) + c->g_bytes + 8ull * c->part_slots +
         4ull * (c->part_slots + 1) + 4ull * c->csr_cap;
}

int launch_solve(fibra_ctx* c, const double* dF, const fibra_law* law,
                 const fibra_relax_cfg* rc, const fibra_stiff_cfg* sc, int want_tangent,
                 fibra_point_result* dres) {
  const int n = c->n_points;
  if (!c->d_entries || !c->variant)
    return set_err(c, FIBRA_E_ARG, "upload_library and bind_points must precede solve");
  // configuration validation (ConfigError propagates: relax.cpp:12-19, network.cpp:55-59,
  // stiffness.cpp:10-13)
  if (!(rc->damping >= 0) || !(rc->tolerance > 0) || rc->max_iterations < 1 ||
      !(rc->dt_safety > 0) || rc->dt_safety > 1 || !(rc->density_scale > 0))
    return set_err(c, FIBRA_E_CONFIG, "invalid RelaxConfig");
  if (rc->energy_check)
    return set_err(c, FIBRA_E_CONFIG,
                   "energy_check is a CPU verification diagnostic; not on the device path");
  if (!(law->ea_scale > 0) || (law->kind == 1 && !(law->nonlinearity > 0)) ||
      (law->kind != 0 && law->kind != 1))
    return set_err(c, FIBRA_E_CONFIG, "invalid FiberLaw");
  if (want_tangent && (!(sc->fd_rel_step > 0) || sc->fd_rel_step >= 1e-2))
    return set_err(c, FIBRA_E_CONFIG, "stiffness fd_rel_step must be in (0, 1e-2)");
  for (int p = 0; p < n; ++p) {
    const DeviceEntry& e = c->entries[c->entry_of_point[p]];
    if (!e.config_ok) return set_err(c, FIBRA_E_CONFIG, e.config_err);
  }
  if (n == 0) return FIBRA_OK;
  int r;
  if ((r = ensure_scratch(c, n))) return r;
  const Variant* v = c->variant;
  KernelFn fn = v->fn[law->kind][c->uniform_ea ? 1 : 0];
  const size_t smem = smem_bytes(c);
  FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  int per_sm = 0;
  FB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, v->T, smem));
  if (per_sm < 1) return set_err(c, FIBRA_E_ARG, "DR kernel does not fit on an SM");
  const int n_solves = want_tangent ? 7 * n : n;
  const int grid = std::min(n_solves, per_sm * c->n_sm);
  const size_t ck = static_cast<size_t>(grid) * 12 * c->ck_stride;
  if (ck > c->ckpt_cap) {
    cudaFree(c->d_ckpt);
    c->d_ckpt = nullptr;
    c->ckpt_cap = 0;
    FB_CUDA(c, cudaMalloc(&c->d_ckpt, ck * sizeof(double)));
    c->ckpt_cap = ck;
  }

  DrParams P;
  P.entries = c->d_entries;
  P.entry_of_point = c->d_entry_of_point;
  P.offsets = c->d_offsets;
  P.u = c->d_state[0];
  P.v = c->d_state[1];
  P.a = c->d_state[2];
  P.f_int = c->d_state[3];
  P.f_damp = c->d_state[4];
  P.mass = c->d_state[5];
  P.inv_mass = c->d_state[6];
  P.t = c->d_state[7];
  P.iters = c->d_iters;
  P.converged = c->d_conv;
  P.solve_F = c->d_solveF;
  P.solve_skip = c->d_skip;
  P.out = c->d_out;
  P.base_flag = c->d_flag;
  P.order = c->d_order;
  P.done_list = c->d_done;
  P.ticket = c->d_ticket;
  P.counters = c->d_counters;
  P.ckpt = c->d_ckpt;
  P.ck_stride = c->ck_stride;
  P.ck_interval = 8;
  P.n_points = n;
  P.n_solves = n_solves;
  P.x_bytes = c->x_bytes;
  P.g_bytes = c->g_bytes;
  P.part_slots = c->part_slots;
  P.csr_cap = c->csr_cap;
  P.reuse_warm = sc ? sc->reuse_warm : 1;
  P.law_buckling_off = law->buckling_off;
  P.ea_scale = law->ea_scale;
  P.nonlinearity = law->nonlinearity;
  P.damping = rc->damping;
  P.tolerance = rc->tolerance;
  P.dt_safety = rc->dt_safety;
  P.density_scale = rc->density_scale;
  P.max_iterations = rc->max_iterations;
  P.phase_prof = nullptr;
  if (getenv("FIBRA_PHASE_PROF")) {  // diagnostics: per-warp phase cycle accumulators
    static unsigned long long* buf = nullptr;
    static size_t cap = 0;
    const size_t need = static_cast<size_t>(grid) * (v->T / 32) * 4;
    if (need > cap) { cudaFree(buf); cudaMalloc(&buf, need * 8); cap = need; }
    cudaMemsetAsync(buf, 0, need * 8, c->stream);
    P.phase_prof = buf;
    c->phase_prof = buf;
    c->phase_prof_n = need;
  }

  cudaStream_t st = c->stream;
  FB_CUDA(c, cudaEventRecord(c->ev[0], st));
  FB_CUDA(c, cudaMemsetAsync(c->d_ticket, 0, 2 * sizeof(int), st));
  FB_CUDA(c, cudaMemsetAsync(c->d_counters, 0, 4 * sizeof(unsigned long long), st));
  const int tb = 128;
  prep_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, sc ? sc->fd_rel_step : 1e-5,
                                                c->d_prep, c->d_solveF, c->d_skip, c->d_flag,
                                                c->d_done, c->sched_mode, c->d_hint, c->d_key);
  FB_CUDA(c, cudaGetLastError());
  rank_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, c->d_key, c->d_order);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[1], st));
  fn<<<grid, v->T, smem, st>>>(P);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[2], st));
  post_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, c->d_prep, c->d_out,
                                                c->d_solveF, dres);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[3], st));
  c->last_solves = n_solves;
  c->last_launches = 4;
  return FIBRA_OK;
}

// packed-node view of one reference FiberNetwork (free-first packing, network.cpp:120-143)
struct PackedNet {
  int N = 0, M = 0, NFN = 0;
  std::vector<double> ref, lump;       // by packed node
  std::vector<int> a, b;               // fiber endpoints as packed nodes
  std::vector<double> l0, ea;
  double max_lump = 0;
  bool ok = true;
  std::string err;
};

PackedNet pack(const fibra_net_desc& d) {
  PackedNet P;
  P.N = d.n_nodes;
  P.M = d.n_fibers;
  P.NFN = d.n_free / 3;
  std::vector<int> node_of_pn(P.N);
  for (int node = 0; node < P.N; ++node) node_of_pn[d.packed_of_dof[3 * node] / 3] = node;
  P.ref.assign(d.packed_ref, d.packed_ref + 3 * static_cast<size_t>(P.N));
  P.lump.resize(P.N);
  for (int pn = 0; pn < P.N; ++pn) {
    P.lump[pn] = d.node_lump[node_of_pn[pn]];
    if (!(P.lump[pn] > 0) && P.ok) {  // setup_mass relax.cpp:29-31
      P.ok = false;
      P.err = "node " + std::to_string(node_of_pn[pn]) + " has no incident fibers (singular mass)";
    }
    P.max_lump = (P.max_lump < P.lump[pn]) ? P.lump[pn] : P.max_lump;
  }
  P.a.resize(P.M);
  P.b.resize(P.M);
  P.l0.assign(d.rest_length, d.rest_length + P.M);
  P.ea.resize(P.M);
  for (int f = 0; f < P.M; ++f) {
    P.a[f] = d.fiber_packed_dofs[6 * f] / 3;
    P.b[f] = d.fiber_packed_dofs[6 * f + 3] / 3;
    P.ea[f] = d.fiber_area[f] * d.fiber_modulus[f];  // FiberNetwork::fiber_ea
  }
  return P;
}

}  // namespace

extern "C" {

int fibra_cuda_device_count(int* n) {
  return cudaGetDeviceCount(n) == cudaSuccess ? FIBRA_OK : FIBRA_E_CUDA;
}

int fibra_cuda_open(int device, fibra_ctx** out) {
  if (!out) return FIBRA_E_ARG;
  auto* c = new fibra_ctx;
  c->device = device;
  auto bail = [&](int code) {
    delete c;
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(FIBRA_E_CUDA);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return bail(FIBRA_E_CUDA);
  if (prop.major < 10) return bail(FIBRA_E_CUDA);  // sm_100a binary only
  c->n_sm = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  if (cudaMalloc(&c->d_ticket, 2 * sizeof(int)) != cudaSuccess) return bail(FIBRA_E_CUDA);
  if (cudaMalloc(&c->d_counters, 4 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(FIBRA_E_CUDA);
  *out = c;
  return FIBRA_OK;
}

int fibra_cuda_close(fibra_ctx* c) {
  if (!c) return FIBRA_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_points(c);
  free_scratch(c);
  free_library(c);
  cudaFree(c->d_ckpt);
  cudaFree(c->d_ticket);
  cudaFree(c->d_counters);
  for (auto& e : c->ev) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return FIBRA_OK;
}

const char* fibra_cuda_last_error(const fibra_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fibra_cuda_set_stream(fibra_ctx* c, void* stream) {
  cudaSetDevice(c->device);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  } else {
    FB_CUDA(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  return FIBRA_OK;
}

int fibra_cuda_upload_library(fibra_ctx* c, const fibra_net_desc* entries, int32_t n) {
  if (!c || !entries || n < 1) return set_err(c, FIBRA_E_CONFIG, "RVE library is empty");
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  free_library(c);
  std::vector<PackedNet> nets;
  nets.reserve(n);
  for (int i = 0; i < n; ++i) {
    const fibra_net_desc& d = entries[i];
    if (d.n_nodes <= 0 || d.n_fibers < 0 || d.n_free % 3 != 0)
      return set_err(c, FIBRA_E_ARG, "malformed library entry " + std::to_string(i));
    nets.push_back(pack(d));
  }
  // one kernel variant for the whole library: the first whose capacity covers every entry
  c->entries.resize(n);
  for (const Variant& v : kVariants) {
    bool ok = true;
    for (int i = 0; i < n && ok; ++i) {
      const PackedNet& P = nets[i];
      ok = build_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), v.T, v.FPT, v.NPT,
                          c->entries[i].sched) &&
           c->entries[i].sched.node_slots * 24 < 65536;
    }
    if (ok) {
      c->variant = &v;
      break;
    }
  }
  if (!c->variant)
    return set_err(c, FIBRA_E_ARG, "RVE too large for the resident kernel variants");
  c->uniform_ea = true;
  for (const PackedNet& P : nets)
    for (int f = 1; f < P.M && c->uniform_ea; ++f) c->uniform_ea = (P.ea[f] == P.ea[0]);
  std::vector<EntryDev> host(n);
  int max_ts = 0, max_gbytes = 0, max_ent = 0;
  for (int i = 0; i < n; ++i) {
    const PackedNet& P = nets[i];
    DeviceEntry& de = c->entries[i];
    const Schedule& S = de.sched;
    de.config_ok = P.ok;
    de.config_err = P.err;
    const int TS = c->variant->NPT * c->variant->T;  // thread slots; dummy x records at TS, TS+1
    const int FS = S.fiber_slots;
    std::vector<int> slot_pn(TS, -1);
    std::vector<double> slot_ref(3 * static_cast<size_t>(TS), 0.0), slot_lump(TS, 1.0);
    for (int sl = 0; sl < S.node_slots; ++sl) {
      const int pn = S.pn_of_slot[sl];
      slot_pn[sl] = pn;
      if (pn < 0) continue;
      for (int k = 0; k < 3; ++k) slot_ref[3 * sl + k] = P.ref[3 * pn + k];
      slot_lump[sl] = P.lump[pn];
    }
    // g*d records: [real: tail (-g*d) and head (+g*d) per fiber, schedule colouring]
    //               [two per dummy fiber slot, bank = lane] [zero record]
    // (all dummies of one lane share a record pair: their values are never read, and within
    //  one store instruction the 16 lanes still hit 16 different banks)
    std::vector<int> dummy_tail(FS, -1), dummy_head(FS, -1);
    for (int fs = 0; fs < FS; ++fs)
      if (S.fiber_of_fslot[fs] < 0) {
        dummy_tail[fs] = S.gd_slots + fs % 16;
        dummy_head[fs] = S.gd_slots + 16 + fs % 16;
      }
    const int zero_rec = S.gd_slots + 32;
    const int gd_total = zero_rec + 1;
    if (24 * gd_total >= 65536)
      return set_err(c, FIBRA_E_ARG, "too many g*d records for 16-bit offsets in entry " + std::to_string(i));
    // CSR by slot, ascending fiber id, padded to even length with the zero record;
    // entry = byte offset of the node's own record of that fiber
    std::vector<std::vector<int>> lists(TS);
    for (int f = 0; f < P.M; ++f) {
      lists[S.slot_of_pn[S.tail_pn[f]]].push_back(f);
      lists[S.slot_of_pn[S.head_pn[f]]].push_back(f);
    }
    int max_pairs = 0;
    for (int sl = 0; sl < TS; ++sl) {
      std::sort(lists[sl].begin(), lists[sl].end());  // reference order (network.cpp:298-303)
      max_pairs = std::max(max_pairs, static_cast<int>((lists[sl].size() + 1) / 2));
    }
    // step-major pairs: pair kp of slot sl at [kp * TS + sl] (coalesced LDS.64 per step)
    std::vector<int> npairs(TS, 0), ent(2 * static_cast<size_t>(max_pairs) * TS, 24 * zero_rec);
    for (int sl = 0; sl < TS; ++sl) {
      const auto& L = lists[sl];
      const int pn = sl < S.node_slots ? S.pn_of_slot[sl] : -1;
      npairs[sl] = static_cast<int>((L.size() + 1) / 2);
      for (size_t i = 0; i < L.size(); ++i) {
        const int f = L[i];
        ent[2 * ((i / 2) * TS + sl) + (i % 2)] =
            24 * (pn == S.tail_pn[f] ? S.rec_tail[f] : S.rec_head[f]);
      }
    }
    std::vector<int> fab(FS), fg(FS), fid(FS, -1);
    std::vector<double> fl0(FS, 0.5), fea(FS, 1.0);
    for (int fs = 0; fs < FS; ++fs) {
      const int f = S.fiber_of_fslot[fs];
      if (f < 0) {  // dummy: unit segment between the two dummy x records
        fab[fs] = (24 * TS) | ((24 * (TS + 1)) << 16);
        fg[fs] = (24 * dummy_tail[fs]) | ((24 * dummy_head[fs]) << 16);
        continue;
      }
      fab[fs] = (24 * S.slot_of_pn[S.tail_pn[f]]) | ((24 * S.slot_of_pn[S.head_pn[f]]) << 16);
      fg[fs] = (24 * S.rec_tail[f]) | ((24 * S.rec_head[f]) << 16);
      fid[fs] = f;
      fl0[fs] = P.l0[f];
      fea[fs] = P.ea[f];
    }
    EntryDev& E = host[i];
    E.n_nodes = P.N;
    E.n_fibers = P.M;
    E.n_free_nodes = P.NFN;
    E.n_fix_nodes = P.N - P.NFN;
    E.f0 = S.f0;
    E.node_slots = S.node_slots;
    E.fiber_slots = FS;
    E.gd_slots = gd_total;
    E.thread_slots = TS;
    E.max_lump = P.max_lump;
    E.max_ea = entries[i].max_ea;
    E.box_volume = 8.0 * entries[i].box_half * entries[i].box_half * entries[i].box_half;
    auto up = [&](auto** dst, const auto& vec) -> int {
      using Tp = typename std::decay_t<decltype(vec)>::value_type;
      Tp* p = nullptr;
      FB_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(vec.size(), 1) * sizeof(Tp)));
      de.allocs.push_back(p);
      if (!vec.empty())
        FB_CUDA(c, cudaMemcpy(p, vec.data(), vec.size() * sizeof(Tp), cudaMemcpyHostToDevice));
      *dst = p;
      return FIBRA_OK;
    };
    int rc;
    if ((rc = up(&E.slot_pn, slot_pn))) return rc;
    if ((rc = up(&E.slot_ref, slot_ref))) return rc;
    if ((rc = up(&E.slot_lump, slot_lump))) return rc;
    if ((rc = up(&E.csr_npairs, npairs))) return rc;
    {
      int* pairs = nullptr;
      if ((rc = up(&pairs, ent))) return rc;
      E.csr_pairs = reinterpret_cast<const int2*>(pairs);
    }
    E.max_pairs = max_pairs;
    if ((rc = up(&E.fib_ab, fab))) return rc;
    if ((rc = up(&E.fib_g, fg))) return rc;
    if ((rc = up(&E.fib_id, fid))) return rc;
    if ((rc = up(&E.fib_l0, fl0))) return rc;
    if ((rc = up(&E.fib_ea, fea))) return rc;
    de.dev = E;
    max_ts = std::max(max_ts, TS);
    max_ent = std::max(max_ent, static_cast<int>(ent.size()));
    const int gb = std::max(24 * gd_total, 8 * (3 * P.N + 3 * P.NFN + P.M));
    max_gbytes = std::max(max_gbytes, gb);
  }
  c->x_bytes = static_cast<int>(align16(24 * static_cast<size_t>(max_ts + 2)));
  c->g_bytes = static_cast<int>(align16(max_gbytes));
  c->part_slots = max_ts;
  c->csr_cap = max_ent;
  c->ck_stride = max_ts;
  FB_CUDA(c, cudaMalloc(&c->d_entries, sizeof(EntryDev) * n));
  FB_CUDA(c, cudaMemcpy(c->d_entries, host.data(), sizeof(EntryDev) * n, cudaMemcpyHostToDevice));
  return FIBRA_OK;
}

int fibra_cuda_bind_points(fibra_ctx* c, const int32_t* entry_of_point, int32_t n) {
  if (!c || n < 0) return FIBRA_E_ARG;
  if (c->entries.empty()) return set_err(c, FIBRA_E_ARG, "upload_library first");
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  free_points(c);
  c->entry_of_point.assign(entry_of_point, entry_of_point + n);
  c->offsets.assign(n + 1, 0);
  for (int p = 0; p < n; ++p) {
    const int e = entry_of_point[p];
    if (e < 0 || e >= static_cast<int>(c->entries.size()))
      return set_err(c, FIBRA_E_CONFIG, "assignment entry out of range");
    c->offsets[p + 1] = c->offsets[p] + 3LL * c->entries[e].dev.n_nodes;
  }
  c->n_points = n;
  const size_t tot = static_cast<size_t>(c->offsets[n]);
  int rc;
  if ((rc = dalloc(c, &c->d_entry_of_point, n))) return rc;
  if ((rc = dalloc(c, &c->d_offsets, n + 1))) return rc;
  for (int k = 0; k < 7; ++k)
    if ((rc = dalloc(c, &c->d_state[k], tot))) return rc;
  if ((rc = dalloc(c, &c->d_state[7], n))) return rc;
  if ((rc = dalloc(c, &c->d_iters, n))) return rc;
  if ((rc = dalloc(c, &c->d_conv, n))) return rc;
  if (n) {
    FB_CUDA(c, cudaMemcpy(c->d_entry_of_point, entry_of_point, sizeof(int) * n, cudaMemcpyHostToDevice));
  }
  FB_CUDA(c, cudaMemcpy(c->d_offsets, c->offsets.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice));
  return fibra_cuda_reset_states(c);
}

int fibra_cuda_set_schedule(fibra_ctx* c, int32_t mode, const double* cost_hint) {
  if (!c) return FIBRA_E_ARG;
  if (mode != FIBRA_SCHED_BATCH && mode != FIBRA_SCHED_STRAIN && mode != FIBRA_SCHED_HINT)
    return set_err(c, FIBRA_E_ARG, "unknown schedule mode");
  if (mode == FIBRA_SCHED_HINT) {
    if (!cost_hint) return set_err(c, FIBRA_E_ARG, "FIBRA_SCHED_HINT needs cost_hint");
    if (c->offsets.empty()) return set_err(c, FIBRA_E_ARG, "bind_points first");
    FB_CUDA(c, cudaSetDevice(c->device));
    FB_CUDA(c, cudaStreamSynchronize(c->stream));
    const size_t n = std::max(c->n_points, 1);
    if (!c->d_hint) {
      int rc;
      if ((rc = dalloc(c, &c->d_hint, n))) return rc;
    }
    if (c->n_points)
      FB_CUDA(c, cudaMemcpy(c->d_hint, cost_hint, sizeof(double) * c->n_points, cudaMemcpyHostToDevice));
  }
  c->sched_mode = mode;
  return FIBRA_OK;
}

int fibra_cuda_reset_states(fibra_ctx* c) {
  FB_CUDA(c, cudaSetDevice(c->device));
  const size_t tot = c->offsets.empty() ? 0 : static_cast<size_t>(c->offsets.back());
  for (int k = 0; k < 7; ++k)
    FB_CUDA(c, cudaMemsetAsync(c->d_state[k], 0, std::max<size_t>(tot, 1) * sizeof(double), c->stream));
  const size_t n = std::max(c->n_points, 1);
  FB_CUDA(c, cudaMemsetAsync(c->d_state[7], 0, n * sizeof(double), c->stream));
  FB_CUDA(c, cudaMemsetAsync(c->d_iters, 0, n * sizeof(long long), c->stream));
  FB_CUDA(c, cudaMemsetAsync(c->d_conv, 0, n, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  return FIBRA_OK;
}

int fibra_cuda_upload_states(fibra_ctx* c, const double* u, const double* t, const int64_t* iters,
                             const uint8_t* converged) {
  FB_CUDA(c, cudaSetDevice(c->device));
  const size_t tot = static_cast<size_t>(c->offsets.back());
  const size_t n = c->n_points;
  if (u && tot) FB_CUDA(c, cudaMemcpyAsync(c->d_state[0], u, tot * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (t && n) FB_CUDA(c, cudaMemcpyAsync(c->d_state[7], t, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (iters && n) FB_CUDA(c, cudaMemcpyAsync(c->d_iters, iters, n * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
  if (converged && n) FB_CUDA(c, cudaMemcpyAsync(c->d_conv, converged, n, cudaMemcpyHostToDevice, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  return FIBRA_OK;
}

int fibra_cuda_download_states(fibra_ctx* c, double* u, double* v, double* a, double* f_int,
                               double* f_damp, double* mass, double* inv_mass, double* t,
                               int64_t* iters, uint8_t* converged) {
  FB_CUDA(c, cudaSetDevice(c->device));
  const size_t tot = static_cast<size_t>(c->offsets.back());
  const size_t n = c->n_points;
  double* dst[7] = {u, v, a, f_int, f_damp, mass, inv_mass};
  for (int k = 0; k < 7; ++k)
    if (dst[k] && tot)
      FB_CUDA(c, cudaMemcpyAsync(dst[k], c->d_state[k], tot * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (t && n) FB_CUDA(c, cudaMemcpyAsync(t, c->d_state[7], n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (iters && n) FB_CUDA(c, cudaMemcpyAsync(iters, c->d_iters, n * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  if (converged && n) FB_CUDA(c, cudaMemcpyAsync(converged, c->d_conv, n, cudaMemcpyDeviceToHost, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  return FIBRA_OK;
}

int fibra_cuda_solve(fibra_ctx* c, const double* F, const fibra_law* law,
                     const fibra_relax_cfg* relax, const fibra_stiff_cfg* stiff,
                     int32_t want_tangent, fibra_point_result* out) {
  if (!c || !law || !relax) return FIBRA_E_ARG;
  FB_CUDA(c, cudaSetDevice(c->device));
  const int n = c->n_points;
  int rc;
  if ((rc = ensure_scratch(c, std::max(n, 1)))) return rc;
  if (n) {
    std::memcpy(c->h_F, F, sizeof(double) * 9 * n);
    FB_CUDA(c, cudaMemcpyAsync(c->d_F, c->h_F, sizeof(double) * 9 * n, cudaMemcpyHostToDevice, c->stream));
  }
  if ((rc = launch_solve(c, c->d_F, law, relax, stiff, want_tangent, c->d_res))) return rc;
  if (n) {
    FB_CUDA(c, cudaMemcpyAsync(c->h_res, c->d_res, sizeof(fibra_point_result) * n,
                               cudaMemcpyDeviceToHost, c->stream));
    FB_CUDA(c, cudaStreamSynchronize(c->stream));
    std::memcpy(out, c->h_res, sizeof(fibra_point_result) * n);
  }
  return FIBRA_OK;
}

int fibra_cuda_solve_device(fibra_ctx* c, const double* F_dev, const fibra_law* law,
                            const fibra_relax_cfg* relax, const fibra_stiff_cfg* stiff,
                            int32_t want_tangent, fibra_point_result* out_dev) {
  if (!c || !law || !relax) return FIBRA_E_ARG;
  FB_CUDA(c, cudaSetDevice(c->device));
  return launch_solve(c, F_dev, law, relax, stiff, want_tangent, out_dev);
}

int fibra_cuda_selftest_fastmath(fibra_ctx* c, uint64_t n, uint64_t seed, uint64_t* mismatches) {
  FB_CUDA(c, cudaSetDevice(c->device));
  unsigned long long* d = nullptr;
  FB_CUDA(c, cudaMalloc(&d, sizeof(unsigned long long)));
  FB_CUDA(c, cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
  fastmath_selftest_kernel<<<4 * c->n_sm, 256, 0, c->stream>>>(n, seed, d);
  FB_CUDA(c, cudaGetLastError());
  unsigned long long h = 0;
  FB_CUDA(c, cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(d);
  *mismatches = h;
  return FIBRA_OK;
}

int fibra_cuda_fp64_peak(fibra_ctx* c, double* out) {
  FB_CUDA(c, cudaSetDevice(c->device));
  double* sink = nullptr;
  FB_CUDA(c, cudaMalloc(&sink, 1024 * sizeof(double)));
  const int iters = 1 << 16, blocks = 4 * c->n_sm, threads = 256;
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  fp64_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink, 64, 1e-9);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {  // best of three, stream otherwise idle
    FB_CUDA(c, cudaEventRecord(c->ev[0], c->stream));
    fp64_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink, iters, 1e-9);
    FB_CUDA(c, cudaEventRecord(c->ev[3], c->stream));
    FB_CUDA(c, cudaEventSynchronize(c->ev[3]));
    float ms = 0;
    FB_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]));
    best = std::min(best, ms);
  }
  cudaFree(sink);
  *out = 8.0 * iters * static_cast<double>(blocks) * threads / (best * 1e-3);
  return FIBRA_OK;
}

int fibra_cuda_phase_profile(fibra_ctx* c, unsigned long long* out, size_t cap, size_t* n) {
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  *n = c->phase_prof_n;
  if (c->phase_prof && out && cap >= c->phase_prof_n)
    FB_CUDA(c, cudaMemcpy(out, c->phase_prof, c->phase_prof_n * 8, cudaMemcpyDeviceToHost));
  return FIBRA_OK;
}

int fibra_cuda_synchronize(fibra_ctx* c) {
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  FB_CUDA(c, cudaGetLastError());
  return FIBRA_OK;
}

int fibra_cuda_last_stats(fibra_ctx* c, fibra_solve_stats* s) {
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  unsigned long long cnt[4] = {0, 0, 0, 0};
  FB_CUDA(c, cudaMemcpy(cnt, c->d_counters, sizeof cnt, cudaMemcpyDeviceToHost));
  std::memset(s, 0, sizeof *s);
  s->iterations = static_cast<int64_t>(cnt[0]);
  s->fiber_iterations = static_cast<int64_t>(cnt[1]);
  s->pipe_ops = static_cast<int64_t>(cnt[2]);
  s->solves = static_cast<int64_t>(cnt[3]);
  float ms = 0;
  if (cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]) == cudaSuccess) s->dr_kernel_ms = ms;
  if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]) == cudaSuccess) s->total_ms = ms;
  s->kernel_launches = c->last_launches;
  return FIBRA_OK;
}

}  // extern "C"
