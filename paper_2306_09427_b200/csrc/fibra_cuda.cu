// B200 batched RVE solver: device context, prep/post kernels and the C-ABI
// (include/fibra_cuda.h).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// --fmad=false -lineinfo (see paper_2306_09427_b200/build.py).
//
// One fibra_cuda_solve == the reference batch_response (proj/src/batch.cpp:155-187) for
// every point:
//   prep_kernel   per point: polar_decompose(F) (tensor.cpp:203-224), probe stretches
//                 U + h T_q (stiffness.cpp:86-127), schedule key; one thread per point;
//                 then a CUB radix sort orders the points longest-expected-first per class
//   DR kernels    one persistent launch per kernel class (resident: dr_kernel.cuh, one RVE
//                 per CTA; cluster: dr_cluster.cuh, one RVE per thread-block cluster), all
//                 DR solves of the class (bases, then probes in base-completion order) from
//                 the class's ticket queue; classes run concurrently on forked streams
//   post_kernel   per point: A from probes (stiffness.cpp:15-41), C = push-forward(A, F)
//                 (tensor.cpp:286-300), sigma = R sigma_U R^T (stiffness.cpp:171-173)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "dr_cluster.cuh"
#include "dr_kernel.cuh"
#include "host/cluster_schedule.hpp"
#include "host/node_schedule.hpp"
#include "host/schedule.hpp"
#include "fibra_cuda.h"
#include "tensor.cuh"
#include "variants.hpp"

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
                            const double* __restrict__ hint, const int* __restrict__ cls,
                            const float* __restrict__ pcost, unsigned* key, int* pidx) {
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
    // input-only cost model: log(expected iterations) = topology term of the entry (upload)
    // - 0.37 log |F^T F - I|; descending (small strain relaxes longest; identity last)
    double e2 = 0;  // |F^T F - I|^2, fp64 only for ordering
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double c = f[i] * f[j] + f[3 + i] * f[3 + j] + f[6 + i] * f[6 + j] - (i == j);
        e2 += c * c;
      }
    const float k = e2 > 0 ? pcost[p] - 0.185f * logf(static_cast<float>(e2)) : -INFINITY;
    if (k == k) {
      const unsigned u = __float_as_uint(k);
      hi = ~((u & 0x80000000u) ? ~u : (u | 0x80000000u));  // descending total order
    } else {
      hi = 0xffffffffu;
    }
  } else if (sched_mode == FIBRA_SCHED_HINT) {
    const float k = static_cast<float>(hint[p]);
    hi = (k == k && k > 0) ? ~__float_as_uint(k) : 0xffffffffu;
  }
  // [kernel class : 4][cost : 28], sorted stably (ties keep point order) -- the order is
  // grouped by class
  key[p] = (static_cast<unsigned>(cls[p]) << 28) | (hi >> 4);
  pidx[p] = p;
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

// orientation_p2 (network.cpp:398-415) of the device-resident state: reference fibre order
// and expression order, one thread per requested point (sequential sums as the reference)
struct OrientDev {
  int n_fibers, pad;
  const int* a;         // [M] packed node of the fibre's end a (fiber_packed_dofs / 3)
  const int* b;         // [M]
  const double* ref;    // [3N] packed reference coordinates
};

__global__ void orientation_kernel(int n, const int* __restrict__ points,
                                   const int* __restrict__ entry_of_point,
                                   const long long* __restrict__ offsets,
                                   const OrientDev* __restrict__ ents, const double* u,
                                   double r0, double r1, double r2, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = points[i];
  const OrientDev& E = ents[entry_of_point[p]];
  const double* up = u + offsets[p];
  const double* ref = E.ref;
  double wsum = 0, acc = 0;
  for (int f = 0; f < E.n_fibers; ++f) {
    const int pa = 3 * E.a[f], pb = 3 * E.b[f];
    const double d0 = (ref[pb] + up[pb]) - (ref[pa] + up[pa]);
    const double d1 = (ref[pb + 1] + up[pb + 1]) - (ref[pa + 1] + up[pa + 1]);
    const double d2 = (ref[pb + 2] + up[pb + 2]) - (ref[pa + 2] + up[pa + 2]);
    const double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (!(len > 0)) continue;
    const double c = (d0 * r0 + d1 * r1 + d2 * r2) / len;
    acc += len * 0.5 * (3.0 * c * c - 1.0);
    wsum += len;
  }
  out[i] = wsum > 0 ? acc / wsum : 0.0;
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
    q = div_fast_i(a, b, ok);  // integer-predicate variant of the DR kernels
    if (!ok) q = a / b;
    local += !same_bits(q, a / b);
    const double zq = (mode == 3 ? 0.0 : a);  // zero numerators through the escape
    q = div_fast_i(zq, b, ok);
    if (!ok) q = zq / b;
    local += !same_bits(q, zq / b);
    local += le_nonneg_bits(fabs(a), fabs(b)) != (fabs(a) <= fabs(b)) && !isnan(a) && !isnan(b);
    const double x = mode == 2 ? a : fabs(a);
    double s = sqrt_fast(x, ok);
    if (!ok) s = sqrt(x);
    local += !same_bits(s, sqrt(x));
  }
  if (local) atomicAdd(bad, local);
}

// expm1 / exp of the exponential fibre law (libm_glibc.cuh) on the device, for the parity
// test against the host libm (tests/test_gpu_fastmath.py)
__global__ void eval_libm_kernel(int which, const double* x, long long n, double* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = which ? glibc::expm1(x[i]) : glibc::exp(x[i]);
}

// (l0, 0) -> (l0, rcp_refined(l0)) for the streaming kernel's incidence rows
__global__ void init_rcp_kernel(double2* p, long long n) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n) p[i].y = rcp_refined(p[i].x);
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
// kernel classes (shapes in variants.hpp, instantiated in kernels_*.cu)
// ---------------------------------------------------------------------------------
constexpr int kMaxClasses = 16;  // 4 bits of the schedule key

struct DeviceEntry {
  EntryDev dev;           // resident-kernel entry
  NodeEntryDev ndev;      // node-centric kernel entry
  StreamEntryDev sdev;    // HBM-streaming kernel entry
  ClusterEntryDev cdev;   // cluster-kernel entry
  OrientDev orient;       // reference-order fibres + packed reference (orientation_p2)
  Schedule sched;
  NodeSchedule nsched;
  std::vector<void*> allocs;
  int cls = -1;           // kernel class
  float log_its = 0;      // topology term of the schedule cost model (upload_library)
  int n_nodes = 0;
  bool config_ok = true;
  std::string config_err;
};

// A kernel class: one kernel shape (resident variant, or cluster variant x cluster size)
// and the library entries it solves.  Each class runs its own persistent launch with its
// own ticket queue; classes of one call run concurrently on forked streams.
struct KClass {
  bool cluster = false;
  bool node = false;      // node-centric resident kernel (dr_node.cuh)
  bool streaming = false; // HBM-streaming cluster kernel (dr_stream.cuh)
  int s_cap = 0, n_cap = 0, m_cap = 0;  // stream: slots, nodes, fibres (scratch layout)
  long long stage_bytes = 0;            // stream: largest per-CTA incidence-row block (entries)
  int vi = 0, C = 1;
  int x_bytes = 0, g_bytes = 0, ts = 0, csr_cap = 0, push_cap = 0, ck_stride = 0;
  int max_halo = 0;  // cluster: halo slots per bank (two banks, dr_cluster.cuh)
  long long scratch_stride = 0;
  bool uniform_ea = true;
  EntryDev* d_entries = nullptr;          // [n_entries] (resident)
  NodeEntryDev* d_nentries = nullptr;     // [n_entries] (node)
  StreamEntryDev* d_sentries = nullptr;   // [n_entries] (stream)
  ClusterEntryDev* d_centries = nullptr;  // [n_entries] (cluster)
  int n_points = 0, point_off = 0;        // bound points of the class, offset in the order
  cudaStream_t stream = nullptr;   // head launch (several classes) or the class's only launch
  cudaStream_t stream2 = nullptr;  // body launch
  cudaEvent_t done = nullptr, done2 = nullptr;
  cudaEvent_t done_t = nullptr;  // timed end of both (FIBRA_CLASS_TIMES diagnostics)
  double* d_ckpt = nullptr;
  size_t ckpt_cap = 0;
  double* d_scratch = nullptr;
  size_t scratch_cap = 0;
  // node classes: x double buffer + incidence tables (x offsets, (l0, 1/l0), EA when not
  // uniform, reduced mass for the nonlinear law)
  size_t node_smem(bool nonlinear) const {
    return 2ull * x_bytes + ((4ull * csr_cap + 15) & ~15ull) + 16ull * csr_cap +
           (uniform_ea ? 0ull : 8ull * csr_cap) + (nonlinear ? 8ull * csr_cap : 0ull);
  }
  long long stream_scratch() const {  // doubles per cluster (dr_stream.cuh layout)
    return 6ll * s_cap + 9ll * n_cap + m_cap + 8 + 2 * 16 * 16;
  }
  size_t smem() const {
    if (streaming) return 0;
    if (node) return node_smem(true);
    if (cluster)
      return static_cast<size_t>(x_bytes) + g_bytes + 8ull * ts + 8ull * csr_cap + 4ull * push_cap;
    return static_cast<size_t>(x_bytes) + g_bytes + 16ull * ts + 4ull * csr_cap;  // dr_kernel.cuh
  }
};

}  // namespace fibra_b200

using namespace fibra_b200;

struct fibra_ctx {
  int device = 0;
  int n_sm = 0;
  int max_smem = 0;  // opt-in dynamic shared memory per block
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  std::string err;
  std::vector<DeviceEntry> entries;
  std::vector<KClass> classes;
  // points
  int n_points = 0;
  std::vector<int32_t> entry_of_point;
  std::vector<long long> offsets;
  int* d_entry_of_point = nullptr;
  float* d_pcost = nullptr;              // per point: the entry's topology term of the cost model
  int* d_class_of_point = nullptr;
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
  unsigned* d_key = nullptr;             // schedule keys, sorted with the point ids by CUB
  unsigned* d_key_sorted = nullptr;
  int* d_pidx = nullptr;
  void* d_sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  fibra_point_result* d_res = nullptr;
  double* h_F = nullptr;                 // pinned staging
  fibra_point_result* h_res = nullptr;   // pinned staging
  int* d_ticket = nullptr;               // [kMaxClasses][2]
  OrientDev* d_orient = nullptr;         // [n_entries]
  unsigned long long* d_counters = nullptr;
  cudaEvent_t ev[4] = {};
  cudaEvent_t ev_fork = nullptr;
  int last_solves = 0;
  int last_launches = 0;
  unsigned long long* phase_prof = nullptr;
  size_t phase_prof_n = 0;
  unsigned long long* d_trace = nullptr;  // FIBRA_TRACE diagnostics: [solve][4]
  size_t trace_cap = 0, trace_n = 0;
  // ---- multi-device context (fibra_cuda_open_devices): one sub-context per device over a
  // shard of the points; this context then holds no device state of its own ----
  std::vector<fibra_ctx*> subs;
  std::vector<ncclComm_t> comms;
  std::vector<double> entry_cost;               // fibra_network_cost per library entry
  std::vector<float> entry_log_its;             // its topology term (schedule cost model)
  std::vector<int> entry_fibers, entry_ndof;
  bool plan_pending = false;                    // bound, shards not yet planned
  bool staged = false;                          // states uploaded before the plan
  std::vector<double> stage_u, stage_t;
  std::vector<int64_t> stage_iters;
  std::vector<uint8_t> stage_conv;
  std::vector<int32_t> dev_of_point, local_of_point;
  std::vector<std::vector<int32_t>> shard;      // global point ids per device, ascending
  int block = 0;                                // records per device block (largest shard)
  std::vector<fibra_point_result*> d_block;     // per device: its block of records
  std::vector<fibra_point_result*> d_gather;    // per device: n_dev blocks (all-gather)
  std::vector<double*> d_Fsh;                   // per device: its shard's F
  std::vector<int32_t*> d_Fidx;                 // device 0: global point ids per shard
  int* d_src = nullptr;                         // device 0: point -> gathered record index
  fibra_point_result* d_out0 = nullptr;         // device 0: records in point order (host path)
  double* d_F0 = nullptr;                       // device 0: F of the host path
  int cap0 = 0;
  float last_gather_ms = 0;
  int host_threads = 0;  // host build threads of upload_library (0: all cores)
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
  cudaFree(c->d_pcost);
  c->d_pcost = nullptr;
  cudaFree(c->d_class_of_point);
  c->d_class_of_point = nullptr;
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
  cudaFree(c->d_key_sorted);
  cudaFree(c->d_pidx);
  cudaFree(c->d_sort_tmp);
  c->d_key_sorted = nullptr;
  c->d_pidx = nullptr;
  c->d_sort_tmp = nullptr;
  c->sort_tmp_bytes = 0;
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
  for (auto& k : c->classes) {
    cudaFree(k.d_entries);
    cudaFree(k.d_nentries);
    cudaFree(k.d_sentries);
    cudaFree(k.d_centries);
    cudaFree(k.d_ckpt);
    cudaFree(k.d_scratch);
    if (k.stream) cudaStreamDestroy(k.stream);
    if (k.stream2) cudaStreamDestroy(k.stream2);
    if (k.done) cudaEventDestroy(k.done);
    if (k.done2) cudaEventDestroy(k.done2);
    if (k.done_t) cudaEventDestroy(k.done_t);
  }
  c->classes.clear();
  cudaFree(c->d_orient);
  c->d_orient = nullptr;
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
  if ((rc = dalloc(c, &c->d_key_sorted, n))) return rc;
  if ((rc = dalloc(c, &c->d_pidx, n))) return rc;
  FB_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, c->sort_tmp_bytes, c->d_key, c->d_key_sorted,
                                             c->d_pidx, c->d_order, n));
  FB_CUDA(c, cudaMalloc(&c->d_sort_tmp, std::max<size_t>(c->sort_tmp_bytes, 1)));
  if ((rc = dalloc(c, &c->d_res, n))) return rc;
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_F), 9 * sizeof(double) * n));
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_res), sizeof(fibra_point_result) * n));
  c->cap_points = n;
  return FIBRA_OK;
}

size_t align16(size_t b) { return (b + 15) & ~static_cast<size_t>(15); }

template <class Tp>
int grow(fibra_ctx* c, Tp** p, size_t& cap, size_t need) {
  if (need <= cap) return FIBRA_OK;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  FB_CUDA(c, cudaMalloc(reinterpret_cast<void**>(p), need * sizeof(Tp)));
  cap = need;
  return FIBRA_OK;
}

int launch_solve(fibra_ctx* c, const double* dF, const fibra_law* law,
                 const fibra_relax_cfg* rc, const fibra_stiff_cfg* sc, int want_tangent,
                 fibra_point_result* dres) {
  const int n = c->n_points;
  if (c->classes.empty() || c->offsets.empty())
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

  DrParams P;
  P.entries = nullptr;
  P.nentries = nullptr;
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
  P.counters = c->d_counters;
  P.ck_interval = kCkInterval;
  P.n_points = n;
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
  P.trace = nullptr;
  cudaStream_t st = c->stream;
  if (getenv("FIBRA_TRACE")) {  // diagnostics: per-solve start/end/SM (fibra_cuda_trace)
    const size_t need = 4ull * (want_tangent ? 7 : 1) * n;
    if (need > c->trace_cap) {
      cudaFree(c->d_trace);
      FB_CUDA(c, cudaMalloc(&c->d_trace, need * 8));
      c->trace_cap = need;
    }
    FB_CUDA(c, cudaMemsetAsync(c->d_trace, 0, need * 8, st));
    P.trace = c->d_trace;
    c->trace_n = need;
  }

  FB_CUDA(c, cudaEventRecord(c->ev[0], st));
  FB_CUDA(c, cudaMemsetAsync(c->d_ticket, 0, 2 * kMaxClasses * sizeof(int), st));
  FB_CUDA(c, cudaMemsetAsync(c->d_counters, 0, 5 * sizeof(unsigned long long), st));
  const int tb = 128;
  prep_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, sc ? sc->fd_rel_step : 1e-5,
                                                c->d_prep, c->d_solveF, c->d_skip, c->d_flag,
                                                c->d_done, c->sched_mode, c->d_hint,
                                                c->d_class_of_point, c->d_pcost, c->d_key,
                                                c->d_pidx);
  FB_CUDA(c, cudaGetLastError());
  size_t tmp_bytes = c->sort_tmp_bytes;  // longest expected solve first, grouped by class
  FB_CUDA(c, cub::DeviceRadixSort::SortPairs(c->d_sort_tmp, tmp_bytes, c->d_key, c->d_key_sorted,
                                             c->d_pidx, c->d_order, n, 0, 32, st));
  FB_CUDA(c, cudaEventRecord(c->ev[1], st));
  FB_CUDA(c, cudaEventRecord(c->ev_fork, st));

  // Classes run concurrently as persistent grids sharing the device.  One full grid per
  // class, launched by descending work, runs the classes nearly back to back (a later
  // launch gets SMs only as earlier grids drain), so each class's longest solves -- 500k
  // iteration caps of 1-2 s -- start only when its turn comes (FIBRA_TRACE timelines,
  // DESIGN.md "Scheduling the batch").  With several classes, each one first gets a "head"
  // launch sized to its share of the estimated work (cost model: sum over its points of
  // exp(log_its) x fibres), so every class's longest-expected solves start at once; then the
  // "body" launches (the rest of each full grid, descending work) fill SMs as heads drain.
  // All launches of a class draw from its one ticket queue.
  std::vector<int> launch_order;
  std::vector<double> class_work(c->classes.size(), 0.0), class_cost(c->classes.size(), 0.0);
  for (int p = 0; p < n; ++p) {
    const DeviceEntry& de = c->entries[c->entry_of_point[p]];
    const KClass& Kc = c->classes[de.cls];
    const int m = Kc.cluster  ? de.cdev.n_fibers
                  : Kc.node   ? de.ndev.n_fibers
                  : Kc.streaming ? de.sdev.n_fibers
                              : de.dev.n_fibers;
    class_work[de.cls] += m;
    class_cost[de.cls] += std::exp(static_cast<double>(de.log_its)) * m;
  }
  double cost_total = 0;
  for (int k = 0; k < static_cast<int>(c->classes.size()); ++k)
    if (c->classes[k].n_points) {
      launch_order.push_back(k);
      cost_total += class_cost[k];
    }
  const char* order_env = getenv("FIBRA_CLASS_ORDER");  // diagnostics: "asc" | "desc"
  const bool ascending = order_env && order_env[0] == 'a';
  std::stable_sort(launch_order.begin(), launch_order.end(), [&](int a, int b) {
    return ascending ? class_work[a] < class_work[b] : class_work[a] > class_work[b];
  });
  const char* heads_env = getenv("FIBRA_CLASS_HEADS");  // diagnostics: "0" = one grid per class
  const bool heads = launch_order.size() > 1 && !(heads_env && heads_env[0] == '0');
  int launches = 2;  // ours: prep and post, plus the DR launches (the sort is CUB's)
  bool prof_used = false;
  // per class: full grid (CTAs, or clusters), head size, kernel handles
  struct Plan {
    int full = 0, head = 0, per_unit = 1;
  };
  std::vector<Plan> plan(c->classes.size());
  for (int ci : launch_order) {
    KClass& K = c->classes[ci];
    const int n_solves = want_tangent ? 7 * K.n_points : K.n_points;
    const size_t smem = K.smem();
    int cap = 0;  // co-resident CTAs (resident) or clusters (cluster) on the device
    if (K.streaming) {
      const StreamVariant& v = kStreamVariants[K.vi];
      StreamFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      if (K.C > 8)
        FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = K.C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      const char* st_env = getenv("FIBRA_STREAM_STAGE");
      const long long sbytes =
          K.stage_bytes * (20 + (K.uniform_ea ? 0 : 8) + (law->kind != 0 ? 8 : 0));
      const bool stage = sbytes <= c->max_smem && !(st_env && st_env[0] == '0');
      const size_t dyn = stage ? static_cast<size_t>(sbytes) : 0;
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(dyn)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(K.C);
      cfg.blockDim = dim3(v.T);
      cfg.dynamicSmemBytes = dyn;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FB_CUDA(c, cudaOccupancyMaxActiveClusters(&cap, fn, &cfg));
      if (cap < 1)
        return set_err(c, FIBRA_E_ARG, "streaming DR kernel cannot be co-scheduled on this device");
    } else if (K.node) {
      const NodeVariant& v = kNodeVariants[K.vi];
      KernelFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      const size_t nsm = K.node_smem(law->kind != 0);
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(nsm)));
      int per_sm = 0;
      FB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, v.T, nsm));
      if (per_sm < 1) return set_err(c, FIBRA_E_ARG, "node DR kernel does not fit on an SM");
      cap = per_sm * c->n_sm;
      plan[ci].per_unit = per_sm;
    } else if (!K.cluster) {
      const Variant& v = kVariants[K.vi];
      KernelFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      int per_sm = 0;
      FB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, v.T, smem));
      if (per_sm < 1) return set_err(c, FIBRA_E_ARG, "DR kernel does not fit on an SM");
      cap = per_sm * c->n_sm;
      plan[ci].per_unit = per_sm;
    } else {
      const ClusterVariant& v = kClusterVariants[K.vi];
      ClusterFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      if (K.C > 8)
        FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = K.C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(K.C);
      cfg.blockDim = dim3(v.T);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FB_CUDA(c, cudaOccupancyMaxActiveClusters(&cap, fn, &cfg));
      if (cap < 1)
        return set_err(c, FIBRA_E_ARG, "cluster DR kernel cannot be co-scheduled on this device");
    }
    plan[ci].full = std::min(n_solves, cap);
    if (heads) {
      const double share = cost_total > 0 ? class_cost[ci] / cost_total : 1.0;
      plan[ci].head = std::max(1, std::min(plan[ci].full, static_cast<int>(std::lround(cap * share))));
    }
  }
  // launch `units` CTAs (resident) or clusters (cluster) of class ci on stream `sm`, using
  // checkpoint / scratch slots from `slot0` on
  auto launch = [&](int ci, int units, int slot0, cudaStream_t sm) -> int {
    KClass& K = c->classes[ci];
    const int n_solves = want_tangent ? 7 * K.n_points : K.n_points;
    P.n_class = K.n_points;
    P.n_solves = n_solves;
    P.trace_class = ci;
    P.shared_queue = heads ? 1 : 0;
    P.order = c->d_order + K.point_off;
    P.done_list = c->d_done + K.point_off;
    P.ticket = c->d_ticket + 2 * ci;
    P.x_bytes = K.x_bytes;
    P.g_bytes = K.g_bytes;
    P.part_slots = K.ts;
    P.csr_cap = K.csr_cap;
    P.ck_stride = K.ck_stride;
    const size_t smem = K.smem();
    if (K.streaming) {
      const StreamVariant& v = kStreamVariants[K.vi];
      StreamFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = K.C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      // incidence rows TMA-staged in shared memory when a CTA's block fits
      // (diagnostics: FIBRA_STREAM_STAGE=0 streams them every pass)
      const char* st_env = getenv("FIBRA_STREAM_STAGE");
      const long long sbytes =
          K.stage_bytes * (20 + (K.uniform_ea ? 0 : 8) + (law->kind != 0 ? 8 : 0));
      const bool stage = sbytes <= c->max_smem && !(st_env && st_env[0] == '0');
      const size_t dyn = stage ? static_cast<size_t>(sbytes) : 0;
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(dyn)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(units * K.C);
      cfg.blockDim = dim3(v.T);
      cfg.dynamicSmemBytes = dyn;
      cfg.stream = sm;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      StreamParams SPm;
      SPm.stage = stage ? 1 : 0;
      SPm.d = P;
      SPm.d.entries = nullptr;
      SPm.d.nentries = nullptr;
      SPm.d.ckpt = K.d_ckpt + static_cast<size_t>(slot0) * K.C * 12 * K.ck_stride;
      SPm.d.phase_prof = nullptr;
      SPm.sentries = K.d_sentries;
      SPm.scratch = K.d_scratch + static_cast<size_t>(slot0) * K.scratch_stride;
      SPm.scratch_stride = K.scratch_stride;
      SPm.s_cap = K.s_cap;
      SPm.n_cap = K.n_cap;
      SPm.m_cap = K.m_cap;
      FB_CUDA(c, cudaLaunchKernelEx(&cfg, fn, SPm));
    } else if (K.node) {
      const NodeVariant& v = kNodeVariants[K.vi];
      KernelFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      const size_t nsm = K.node_smem(law->kind != 0);
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(nsm)));
      P.first_wave_sms = (!heads && plan[ci].per_unit == 2 && units == 2 * c->n_sm) ? c->n_sm : 0;
      P.entries = nullptr;
      P.nentries = K.d_nentries;
      P.ckpt = K.d_ckpt + static_cast<size_t>(slot0) * 12 * K.ck_stride;
      P.phase_prof = nullptr;
      fn<<<units, v.T, nsm, sm>>>(P);
    } else if (!K.cluster) {
      const Variant& v = kVariants[K.vi];
      KernelFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      // (several classes may share a kernel function: its shared-memory limit is set per launch)
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      P.first_wave_sms = (!heads && plan[ci].per_unit == 2 && units == 2 * c->n_sm) ? c->n_sm : 0;
      P.entries = K.d_entries;
      P.ckpt = K.d_ckpt + static_cast<size_t>(slot0) * 12 * K.ck_stride;
      P.phase_prof = nullptr;
      if (getenv("FIBRA_PHASE_PROF") && !prof_used) {  // diagnostics: per-warp phase cycles
        static unsigned long long* buf = nullptr;
        static size_t pcap = 0;
        const size_t need = static_cast<size_t>(units) * (v.T / 32) * 8;
        if (need > pcap) { cudaFree(buf); cudaMalloc(&buf, need * 8); pcap = need; }
        cudaMemsetAsync(buf, 0, need * 8, sm);
        P.phase_prof = buf;
        c->phase_prof = buf;
        c->phase_prof_n = need;
        prof_used = true;
      }
      fn<<<units, v.T, smem, sm>>>(P);
    } else {
      const ClusterVariant& v = kClusterVariants[K.vi];
      ClusterFn fn = v.fn[law->kind + 2 * (law->buckling_off ? 1 : 0)][K.uniform_ea ? 1 : 0];
      FB_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = K.C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(units * K.C);
      cfg.blockDim = dim3(v.T);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = sm;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      ClusterParams CP;
      CP.d = P;
      CP.d.entries = nullptr;
      CP.d.ckpt = K.d_ckpt + static_cast<size_t>(slot0) * K.C * 12 * K.ck_stride;
      CP.d.phase_prof = nullptr;
      CP.centries = K.d_centries;
      CP.scratch = K.d_scratch + static_cast<size_t>(slot0) * K.scratch_stride;
      CP.scratch_stride = K.scratch_stride;
      CP.push_cap = K.push_cap;
      CP.halo_stride = 24 * K.max_halo;
      CP.debug_no_local = getenv("FIBRA_CLUSTER_NO_LOCAL") ? 1 : 0;
      CP.pad = 0;
      FB_CUDA(c, cudaLaunchKernelEx(&cfg, fn, CP));
    }
    FB_CUDA(c, cudaGetLastError());
    ++launches;
    return FIBRA_OK;
  };
  for (int ci : launch_order) {  // checkpoint / scratch slots for the class's full grid
    KClass& K = c->classes[ci];
    const size_t units = static_cast<size_t>(plan[ci].full);
    if ((r = grow(c, &K.d_ckpt, K.ckpt_cap,
                  units * ((K.cluster || K.streaming) ? K.C : 1) * 12 * K.ck_stride)))
      return r;
    if ((K.cluster || K.streaming) &&
        (r = grow(c, &K.d_scratch, K.scratch_cap, units * K.scratch_stride)))
      return r;
    FB_CUDA(c, cudaStreamWaitEvent(K.stream, c->ev_fork, 0));
    FB_CUDA(c, cudaStreamWaitEvent(K.stream2, c->ev_fork, 0));
  }
  if (heads) {
    std::vector<int> by_cost = launch_order;
    std::stable_sort(by_cost.begin(), by_cost.end(),
                     [&](int a, int b) { return class_cost[a] > class_cost[b]; });
    for (int ci : by_cost)
      if ((r = launch(ci, plan[ci].head, 0, c->classes[ci].stream))) return r;
  }
  for (int ci : launch_order) {
    KClass& K = c->classes[ci];
    const int head = heads ? plan[ci].head : 0;
    if (plan[ci].full > head && (r = launch(ci, plan[ci].full - head, head, K.stream2))) return r;
    FB_CUDA(c, cudaEventRecord(K.done, K.stream));
    FB_CUDA(c, cudaEventRecord(K.done2, K.stream2));
    FB_CUDA(c, cudaStreamWaitEvent(K.stream2, K.done, 0));
    FB_CUDA(c, cudaEventRecord(K.done_t, K.stream2));
    FB_CUDA(c, cudaStreamWaitEvent(st, K.done2, 0));
    FB_CUDA(c, cudaStreamWaitEvent(st, K.done, 0));
  }
  FB_CUDA(c, cudaEventRecord(c->ev[2], st));
  post_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, c->d_prep, c->d_out,
                                                c->d_solveF, dres);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[3], st));
  c->last_solves = want_tangent ? 7 * n : n;
  c->last_launches = launches;
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

// Input-only schedule cost model, topology term: floppy networks (many nodes of degree <= 2,
// few fibres per node) relax slowest; fitted on config-3 knn networks (Spearman 0.83 on
// held-out points vs 0.08 for strain alone, tools/trace_solve.py); only orders / places work
float topology_log_its(const PackedNet& P) {
  std::vector<int> deg(P.N, 0);
  for (int f = 0; f < P.M; ++f) ++deg[P.a[f]], ++deg[P.b[f]];
  int low = 0;
  for (int d : deg) low += d <= 2;
  const double fd2 = P.N ? static_cast<double>(low) / P.N : 0.0;
  const double r = P.N ? static_cast<double>(P.M) / P.N : 0.0;
  return static_cast<float>(7.2 * fd2 - 3.3 * r + 1.75 * std::log(std::max(P.M, 1)));
}

// largest CSR list of a network in entry pairs (incident fibers per node, padded to even)
int max_pairs_of(const PackedNet& P) {
  std::vector<int> deg(P.N, 0);
  for (int f = 0; f < P.M; ++f) {
    ++deg[P.a[f]];
    ++deg[P.b[f]];
  }
  int m = 0;
  for (int pn = 0; pn < P.N; ++pn) m = std::max(m, (deg[pn] + 1) / 2);
  return m;
}

bool resident_fits(const fibra_ctx* c, const PackedNet& P, const Variant& v, int max_pairs,
                   Schedule& S) {
  if (!build_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), v.T, v.FPT, v.NPT, S))
    return false;
  const int TS = v.NPT * v.T;
  const int gd_total = S.gd_slots + 17;  // + per-lane dummy records + the zero record
  if (S.node_slots * 24 >= 65536) return false;  // 16-bit x-record offsets
  const size_t smem = align16(24 * static_cast<size_t>(TS + 32)) +
                      align16(std::max<size_t>(24ull * gd_total, 8ull * (3 * P.N + 3 * P.NFN + P.M))) +
                      16ull * TS + 8ull * (max_pairs + 2) * TS;
  return smem <= static_cast<size_t>(c->max_smem);
}

// the cluster kernel's static control block beyond the common 4 KB reserve
// (the kernel's only static shared memory)
constexpr int kClusterCtlExtra = sizeof(ClusterCtl) > 4096 ? static_cast<int>(sizeof(ClusterCtl)) - 4096 : 0;

// Halo x banks: two (by pass parity) in mirror mode, whose fiber -> node handoff is a CTA
// barrier; one otherwise.  A class's bank stride is 24 x its largest mirror-mode halo
// (Caps::max_halo), and every mirror entry's x region holds two banks of that entry's halo,
// so the class's x region (the per-entry maximum) holds both banks of every mirror entry.
int halo_banks(const ClusterPlan& plan) { return plan.mirror ? 2 : 1; }

size_t cluster_smem(const ClusterPlan& plan, const ClusterVariant& v, int max_pairs) {
  const int TS = v.NPT * v.T;
  size_t max_h = 0;
  for (const ClusterPart& q : plan.parts) max_h = std::max(max_h, q.h_fiber.size());
  return align16(24ull * (TS + 2 + halo_banks(plan) * plan.max_halo)) +
         align16(24ull * (v.FPT * (v.T - 32) + max_h + 1)) + 8ull * TS +
         8ull * max_pairs * TS + 4ull * plan.max_push * TS;
}

bool cluster_fits(const fibra_ctx* c, const PackedNet& P, const ClusterVariant& v, int C,
                  int max_pairs, ClusterPlan& plan) {
  // mirror mode first (one cluster barrier per iteration), else copies of remote records
  // (diagnostics: FIBRA_CLUSTER_MIRROR=0 disables mirror mode)
  const char* me = getenv("FIBRA_CLUSTER_MIRROR");
  const bool try_mirror = !(me && me[0] == '0');
  if (!(try_mirror && build_cluster_plan(P.N, P.NFN, P.M, P.a.data(), P.b.data(), P.ref.data(),
                                         C, v.T, v.FPT, v.NPT, true, plan)) &&
      !build_cluster_plan(P.N, P.NFN, P.M, P.a.data(), P.b.data(), P.ref.data(), C, v.T, v.FPT,
                          v.NPT, false, plan))
    return false;
  const int TS = v.NPT * v.T;
  if (24 * (TS + 2 + plan.max_halo) >= 65536) return false;  // 16-bit x offsets
  return cluster_smem(plan, v, max_pairs) <= static_cast<size_t>(c->max_smem - kClusterCtlExtra);
}

// Host image of one library entry's device arrays: built without CUDA calls (so entries
// are built in parallel), then committed with one allocation and one copy.
struct Arena {
  std::vector<unsigned char> host;
  std::vector<std::pair<void*, size_t>> fixes;  // device pointer fields -> arena offsets
  size_t reserve(size_t bytes) {
    const size_t off = (host.size() + 15) & ~static_cast<size_t>(15);
    host.resize(off + std::max<size_t>(bytes, 16));
    return off;
  }
  template <class Vec, class Tp>
  void add(Tp** dst, const Vec& vec) {
    using Ep = typename Vec::value_type;
    const size_t off = reserve(vec.size() * sizeof(Ep));
    if (!vec.empty()) std::memcpy(host.data() + off, vec.data(), vec.size() * sizeof(Ep));
    fixes.push_back({static_cast<void*>(dst), off});
  }
};

// kernel-class capacities one entry needs (merged into its KClass after the parallel build)
struct Caps {
  int ts = 0, x_bytes = 0, g_bytes = 0, csr_cap = 0, push_cap = 0, max_halo = 0;
  int s_cap = 0, n_cap = 0, m_cap = 0;  // streaming kernel
  long long stage_bytes = 0;
  long long scratch_stride = 0;
};

void merge_caps(KClass& K, const Caps& e) {
  K.ts = e.ts;
  K.ck_stride = e.ts;
  K.x_bytes = std::max(K.x_bytes, e.x_bytes);
  K.g_bytes = std::max(K.g_bytes, e.g_bytes);
  K.csr_cap = std::max(K.csr_cap, e.csr_cap);
  K.push_cap = std::max(K.push_cap, e.push_cap);
  K.max_halo = std::max(K.max_halo, e.max_halo);
  K.scratch_stride = std::max(K.scratch_stride, e.scratch_stride);
  K.s_cap = std::max(K.s_cap, e.s_cap);
  K.n_cap = std::max(K.n_cap, e.n_cap);
  K.m_cap = std::max(K.m_cap, e.m_cap);
  K.stage_bytes = std::max(K.stage_bytes, e.stage_bytes);
  if (K.streaming) K.scratch_stride = K.stream_scratch();
}

// node-centric kernel: shared-memory components of an entry for shape v (Caps fields:
// x_bytes = one x buffer, csr_cap = incidence entries); the footprint is checked for the
// nonlinear law (the largest) and must hold the exit scratch (f, x, m v^2, strain energy).
int node_search_moves() {
  const char* e = getenv("FIBRA_NODE_SEARCH");  // diagnostics: placement search moves
  return e ? atoi(e) : 20000;
}

bool node_fits(const fibra_ctx* c, const PackedNet& P, const NodeVariant& v, bool uniform_ea,
               NodeSchedule& S) {
  const int TS = v.NPT * v.T;
  if (P.N > TS || 24 * TS >= 65536) return false;  // 16-bit x offsets
  if (!build_node_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), v.T, v.NPT,
                           node_search_moves(), S))
    return false;
  KClass K;
  K.node = true;
  K.uniform_ea = uniform_ea;
  K.x_bytes = static_cast<int>(align16(24ull * TS));
  K.csr_cap = 32 * std::max(S.n_rows, 1);
  const size_t region = K.node_smem(false) - 2ull * K.x_bytes;
  const size_t exit_need = 8ull * (3 * P.N + 3 * P.NFN + P.M);
  if (region < exit_need) K.csr_cap = static_cast<int>((exit_need + 19) / 20 + 32);
  return K.node_smem(true) <= static_cast<size_t>(c->max_smem);
}

// node-kernel entry: slot arrays and the step-major incidence tables
void build_node_entry(DeviceEntry& de, const PackedNet& P, const fibra_net_desc& d,
                      const NodeVariant& v, Arena& A, Caps& K) {
  const NodeSchedule& S = de.nsched;
  const int TS = v.NPT * v.T;
  const int G = TS / 32;
  std::vector<int> slot_pn(TS, -1), slot_deg(TS, 0);
  std::vector<double> slot_ref(3 * static_cast<size_t>(TS), 0.0), slot_lump(TS, 1.0);
  for (int sl = 0; sl < TS; ++sl) {
    const int pn = S.pn_of_slot[sl];
    slot_pn[sl] = pn;
    slot_deg[sl] = S.deg[sl];
    if (pn < 0) continue;
    for (int k = 0; k < 3; ++k) slot_ref[3 * sl + k] = P.ref[3 * pn + k];
    slot_lump[sl] = P.lump[pn];
  }
  const size_t ninc = 32ull * S.n_rows;
  std::vector<int> inc_x(ninc, 0);
  std::vector<double> inc_l0(ninc, 1.0), inc_ea(ninc, 1.0), inc_lump(ninc, 1.0);
  for (int g = 0; g < G; ++g)
    for (int l = 0; l < 32; ++l) {
      const int sl = 32 * g + l;
      for (int st = 0; st < S.deg[sl]; ++st) {
        const size_t ix = 32ull * (S.group_row0[g] + st) + l;
        const int f = S.inc_fiber[sl][st], o = S.inc_other[sl][st];
        inc_x[ix] = 24 * S.slot_of_pn[o];
        inc_l0[ix] = P.l0[f];
        inc_ea[ix] = P.ea[f];
        inc_lump[ix] = P.lump[o];
      }
    }
  NodeEntryDev& E = de.ndev;
  E = NodeEntryDev{};
  E.n_nodes = P.N;
  E.n_fibers = P.M;
  E.n_free_nodes = P.NFN;
  E.n_fix_nodes = P.N - P.NFN;
  E.f0 = S.f0;
  E.node_slots = TS;
  E.n_rows = S.n_rows;
  E.max_lump = P.max_lump;
  E.max_ea = d.max_ea;
  E.box_volume = 8.0 * d.box_half * d.box_half * d.box_half;
  A.add(&E.slot_pn, slot_pn);
  A.add(&E.slot_ref, slot_ref);
  A.add(&E.slot_lump, slot_lump);
  A.add(&E.slot_deg, slot_deg);
  A.add(&E.group_row0, S.group_row0);
  A.add(&E.inc_x, inc_x);
  A.add(&E.inc_l0, inc_l0);
  A.add(&E.inc_ea, inc_ea);
  A.add(&E.inc_lump, inc_lump);
  A.add(&E.fib_a, P.a);
  A.add(&E.fib_b, P.b);
  A.add(&E.fib_l0, P.l0);
  A.add(&E.fib_ea, P.ea);
  K.ts = TS;
  K.x_bytes = static_cast<int>(align16(24ull * TS));
  K.csr_cap = 32 * std::max(S.n_rows, 1);
  const size_t region = 2ull * 0 + ((4ull * K.csr_cap + 15) & ~15ull) + 16ull * K.csr_cap;
  const size_t exit_need = 8ull * (3 * P.N + 3 * P.NFN + P.M);
  if (region < exit_need) K.csr_cap = static_cast<int>((exit_need + 19) / 20 + 32);
}

// streaming-kernel entry (dr_stream.cuh): node placement over the cluster's C*T*NPT slots
// (no bank search: the rows and x live in global memory), step-major incidence rows
void build_stream_entry(DeviceEntry& de, const PackedNet& P, const fibra_net_desc& d,
                        const StreamVariant& v, int C, Arena& A, Caps& K) {
  const NodeSchedule& S = de.nsched;
  const int TS = C * v.T * v.NPT;
  const int G = TS / 32;
  std::vector<int> slot_pn(TS, -1), slot_deg(TS, 0);
  std::vector<double> slot_ref(3 * static_cast<size_t>(TS), 0.0), slot_lump(TS, 1.0);
  for (int sl = 0; sl < TS; ++sl) {
    const int pn = S.pn_of_slot[sl];
    slot_pn[sl] = pn;
    slot_deg[sl] = S.deg[sl];
    if (pn < 0) continue;
    for (int k = 0; k < 3; ++k) slot_ref[3 * sl + k] = P.ref[3 * pn + k];
    slot_lump[sl] = P.lump[pn];
  }
  const size_t ninc = 32ull * std::max(S.n_rows, 1);
  std::vector<int> inc_x(ninc, 0);
  std::vector<double> inc_l0(2 * ninc, 1.0), inc_ea(ninc, 1.0), inc_lump(ninc, 1.0);
  for (int g = 0; g < G; ++g)
    for (int l = 0; l < 32; ++l) {
      const int sl = 32 * g + l;
      for (int st = 0; st < S.deg[sl]; ++st) {
        const size_t ix = 32ull * (S.group_row0[g] + st) + l;
        const int f = S.inc_fiber[sl][st], o = S.inc_other[sl][st];
        inc_x[ix] = 3 * S.slot_of_pn[o];
        inc_l0[2 * ix] = P.l0[f];
        inc_l0[2 * ix + 1] = 0.0;  // rcp_refined(l0), filled on the device (init_rcp_kernel)
        inc_ea[ix] = P.ea[f];
        inc_lump[ix] = P.lump[o];
      }
    }
  StreamEntryDev& E = de.sdev;
  E = StreamEntryDev{};
  E.n_nodes = P.N;
  E.n_fibers = P.M;
  E.n_free_nodes = P.NFN;
  E.n_fix_nodes = P.N - P.NFN;
  E.f0 = S.f0;
  E.node_slots = TS;
  E.n_rows = S.n_rows;
  E.max_lump = P.max_lump;
  E.max_ea = d.max_ea;
  E.box_volume = 8.0 * d.box_half * d.box_half * d.box_half;
  E.ea0 = P.M > 0 ? P.ea[0] : 1.0;
  A.add(&E.slot_pn, slot_pn);
  A.add(&E.slot_ref, slot_ref);
  A.add(&E.slot_lump, slot_lump);
  A.add(&E.slot_deg, slot_deg);
  A.add(&E.group_row0, S.group_row0);
  A.add(&E.inc_x, inc_x);
  A.add(reinterpret_cast<const double**>(&E.inc_l0), inc_l0);
  A.add(&E.inc_ea, inc_ea);
  A.add(&E.inc_lump, inc_lump);
  A.add(&E.fib_a, P.a);
  A.add(&E.fib_b, P.b);
  A.add(&E.fib_l0, P.l0);
  A.add(&E.fib_ea, P.ea);
  K.ts = v.T * v.NPT;  // checkpoint slots per CTA
  // incidence entries of one CTA's rows (staged in shared memory at 20 bytes an entry --
  // x offset, l0 pair -- plus EA / lumping weight when the launch needs them), the largest
  // over the cluster's CTAs
  long long stage = 0;
  for (int r = 0; r < C; ++r) {
    long long b = 0;
    for (int j = 0; j < v.NPT; ++j) {
      const int g0 = (j * C * v.T + r * v.T) / 32;
      b += 32ll * (S.group_row0[g0 + v.T / 32] - S.group_row0[g0]);
    }
    stage = std::max(stage, b);
  }
  K.stage_bytes = stage;
  K.s_cap = TS;
  K.n_cap = P.N;
  K.m_cap = P.M;
}

// resident-kernel entry: slot arrays, g*d record colouring, step-major CSR pairs
void build_resident_entry(DeviceEntry& de, const PackedNet& P, const fibra_net_desc& d,
                          const Variant& v, Arena& A, Caps& K) {
  const Schedule& S = de.sched;
  const int TS = v.NPT * v.T;  // thread slots; dummy x records at TS .. TS+31
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
  // g*d records: [real: +g*d per fiber, schedule colouring] [16 dummy records, one per
  // bank] [zero record].  Dummy fibers (empty fiber slots) load x from dummy records too:
  // 16 tail records at slots TS .. TS+15 (0,0,0) and 16 head records at TS+16 .. TS+31
  // (1,0,0), a unit segment.  In each half-warp group a dummy takes x records and a g*d
  // record in banks the group's real fibers leave free, so it adds no bank conflict to the
  // group's loads and stores (values of dummies are never read).
  std::vector<int> dummy_rec(FS, -1), dummy_xt(FS, -1), dummy_xh(FS, -1);
  {
    auto xbank = [](int slot) { return (3 * slot) % 16; };  // 24-byte records: bank pair 3r
    int xt_of_bank[16], xh_of_bank[16], rec_of_bank[16];
    for (int r = 0; r < 16; ++r) {
      xt_of_bank[xbank(TS + r)] = TS + r;
      xh_of_bank[xbank(TS + 16 + r)] = TS + 16 + r;
      rec_of_bank[(3 * (S.gd_slots + r)) % 16] = S.gd_slots + r;
    }
    for (int g = 0; g < FS / 16; ++g) {
      bool ut[16] = {}, uh[16] = {}, ur[16] = {};
      for (int l = 0; l < 16; ++l) {
        const int f = S.fiber_of_fslot[16 * g + l];
        if (f < 0) continue;
        ut[xbank(S.slot_of_pn[S.tail_pn[f]])] = true;
        uh[xbank(S.slot_of_pn[S.head_pn[f]])] = true;
        ur[(3 * S.rec[f]) % 16] = true;
      }
      int bt = 0, bh = 0, br = 0;
      for (int l = 0; l < 16; ++l) {
        const int fs = 16 * g + l;
        if (S.fiber_of_fslot[fs] >= 0) continue;
        while (ut[bt]) ++bt;
        while (uh[bh]) ++bh;
        while (ur[br]) ++br;
        dummy_xt[fs] = xt_of_bank[bt];
        dummy_xh[fs] = xh_of_bank[bh];
        dummy_rec[fs] = rec_of_bank[br];
        ut[bt] = uh[bh] = ur[br] = true;
      }
    }
  }
  const int zero_rec = S.gd_slots + 16;
  const int gd_total = zero_rec + 1;
  // CSR by slot, ascending fiber id, padded to even length with the zero record;
  // entry = byte offset of the fiber's record | 1u << 31 when the node is the fiber's tail
  // (the gather adds -1 * record: f - g*d, network.cpp:298-303)
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
  // step-major pairs: pair kp of slot sl at [kp * TS + sl] (coalesced LDS.64 per step), plus
  // two padding rows of zero-record pairs (the gather loads pairs ahead)
  std::vector<int> npairs(TS, 0), ent(2 * static_cast<size_t>(max_pairs + 2) * TS, 24 * zero_rec);
  for (int sl = 0; sl < TS; ++sl) {
    const auto& L = lists[sl];
    const int pn = sl < S.node_slots ? S.pn_of_slot[sl] : -1;
    npairs[sl] = static_cast<int>((L.size() + 1) / 2);
    for (size_t i = 0; i < L.size(); ++i) {
      const int f = L[i];
      const unsigned neg = pn == S.tail_pn[f] ? 0x80000000u : 0u;
      ent[2 * ((i / 2) * TS + sl) + (i % 2)] = static_cast<int>((24u * S.rec[f]) | neg);
    }
  }
  std::vector<int> fab(FS), fg(FS), fid(FS, -1);
  std::vector<double> fl0(FS, 0.5), fea(FS, P.M > 0 ? P.ea[0] : 1.0);
  for (int fs = 0; fs < FS; ++fs) {
    const int f = S.fiber_of_fslot[fs];
    if (f < 0) {  // dummy: unit segment between two dummy x records
      fab[fs] = (24 * dummy_xt[fs]) | ((24 * dummy_xh[fs]) << 16);
      fg[fs] = 24 * dummy_rec[fs];
      continue;
    }
    fab[fs] = (24 * S.slot_of_pn[S.tail_pn[f]]) | ((24 * S.slot_of_pn[S.head_pn[f]]) << 16);
    fg[fs] = 24 * S.rec[f];
    fid[fs] = f;
    fl0[fs] = P.l0[f];
    fea[fs] = P.ea[f];
  }
  EntryDev& E = de.dev;
  E = EntryDev{};
  E.n_nodes = P.N;
  E.n_fibers = P.M;
  E.n_free_nodes = P.NFN;
  E.n_fix_nodes = P.N - P.NFN;
  E.f0 = S.f0;
  E.node_slots = S.node_slots;
  E.fiber_slots = FS;
  E.gd_slots = gd_total;
  E.thread_slots = TS;
  E.max_pairs = max_pairs;
  E.max_lump = P.max_lump;
  E.max_ea = d.max_ea;
  E.box_volume = 8.0 * d.box_half * d.box_half * d.box_half;
  A.add(&E.slot_pn, slot_pn);
  A.add(&E.slot_ref, slot_ref);
  A.add(&E.slot_lump, slot_lump);
  A.add(&E.csr_npairs, npairs);
  A.add(&E.csr_pairs, ent);
  A.add(&E.fib_ab, fab);
  A.add(&E.fib_g, fg);
  A.add(&E.fib_id, fid);
  A.add(&E.fib_l0, fl0);
  A.add(&E.fib_ea, fea);
  K.ts = TS;
  K.x_bytes = static_cast<int>(align16(24 * static_cast<size_t>(TS + 32)));
  const size_t gb = std::max<size_t>(24ull * gd_total, 8ull * (3 * P.N + 3 * P.NFN + P.M));
  K.g_bytes = static_cast<int>(align16(gb));
  K.csr_cap = static_cast<int>(ent.size());
}

// cluster-kernel entry: one PartDev per CTA (host/cluster_schedule.hpp)
void build_cluster_entry(DeviceEntry& de, const PackedNet& P, const fibra_net_desc& d,
                         const ClusterPlan& plan, const ClusterVariant& v, Arena& A,
                         std::vector<PartDev>& parts, size_t& parts_off, Caps& K) {
  const int C = plan.C, T = v.T, TS = v.NPT * v.T, FS = v.FPT * v.T, FT = T - 32;
  std::vector<std::vector<int>> inc(P.N);  // incident fibers per node, ascending id
  for (int f = 0; f < P.M; ++f) {
    inc[P.a[f]].push_back(f);
    if (P.b[f] != P.a[f]) inc[P.b[f]].push_back(f);
  }
  // per part: record (= compact fiber slot) and plan index of every fiber it evaluates (a
  // mirrored cross fiber has one in each of its two parts), copy index of remote records
  std::vector<std::vector<int>> own_k(C, std::vector<int>(P.M, -1)), own_i(C, std::vector<int>(P.M, -1));
  std::vector<int> hrec(P.M, -1);
  for (int q = 0; q < C; ++q) {
    const ClusterPart& Q = plan.parts[q];
    for (size_t k = 0; k < Q.slot_fiber.size(); ++k)
      if (Q.slot_fiber[k] >= 0) {
        own_k[q][Q.fibers[Q.slot_fiber[k]]] = static_cast<int>(k);
        own_i[q][Q.fibers[Q.slot_fiber[k]]] = Q.slot_fiber[k];
      }
    for (size_t h = 0; h < Q.h_fiber.size(); ++h) hrec[Q.h_fiber[h]] = static_cast<int>(h);
  }
  // halo slot of a remote node in part q, and the push lists of the owners
  std::vector<std::vector<int>> halo_of(C, std::vector<int>());
  std::vector<std::vector<std::vector<int>>> push(C, std::vector<std::vector<int>>(TS));
  for (int q = 0; q < C; ++q) {
    const ClusterPart& Q = plan.parts[q];
    halo_of[q].assign(P.N, -1);
    for (size_t h = 0; h < Q.halo_pn.size(); ++h) {
      const int pn = Q.halo_pn[h];
      halo_of[q][pn] = static_cast<int>(h);
      const int o = plan.part_of_pn[pn];
      push[o][plan.slot_of_pn[pn]].push_back((q << 16) | (24 * (TS + 2 + static_cast<int>(h))));
    }
  }
  parts.assign(C, PartDev{});
  int max_pairs_all = 0, max_push_all = 0, max_rec = 0;
  for (int q = 0; q < C; ++q) {
    const ClusterPart& Q = plan.parts[q];
    PartDev& D = parts[q];
    D = PartDev{};
    const int n_h = static_cast<int>(Q.h_fiber.size());
    // records: [one per fiber slot of the fiber threads, compact index k = j*FT + tid (dummy
    // slots included, so the kernel derives the offset)][copies of remote fibers (heads
    // here)][zero record]
    const int own_slots = v.FPT * FT;
    const int zero_rec = own_slots + n_h;
    std::vector<int> slot_pn(TS, -1);
    std::vector<double> slot_ref(3 * static_cast<size_t>(TS), 0.0), slot_lump(TS, 1.0);
    for (int sl = 0; sl < Q.node_slots; ++sl) {
      const int pn = Q.pn_of_slot[sl];
      slot_pn[sl] = pn;
      if (pn < 0) continue;
      for (int k = 0; k < 3; ++k) slot_ref[3 * sl + k] = P.ref[3 * pn + k];
      slot_lump[sl] = P.lump[pn];
    }
    // CSR: ascending fiber id; the owned fiber's record (negated for its tail) or the copy
    // of a remote fiber's record (this node is its head)
    int max_pairs = 0, max_push = 0;
    std::vector<std::vector<int>> lists(TS);
    for (int sl = 0; sl < Q.node_slots; ++sl) {
      const int pn = Q.pn_of_slot[sl];
      if (pn < 0) continue;
      for (int f : inc[pn]) {
        int e;
        if (own_k[q][f] >= 0) {  // evaluated here
          e = 24 * own_k[q][f];
          if (Q.tail_pn[own_i[q][f]] == pn) e |= static_cast<int>(0x80000000u);
        } else {
          e = 24 * (own_slots + hrec[f]);
        }
        lists[sl].push_back(e);
      }
      max_pairs = std::max(max_pairs, static_cast<int>((lists[sl].size() + 1) / 2));
      max_push = std::max(max_push, static_cast<int>(push[q][sl].size()));
    }
    std::vector<int> npairs(TS, 0), ent(2 * static_cast<size_t>(max_pairs) * TS, 24 * zero_rec);
    std::vector<int> npush(TS, 0), pdst(static_cast<size_t>(max_push) * TS, 0);
    for (int sl = 0; sl < TS; ++sl) {
      const auto& L = lists[sl];
      npairs[sl] = static_cast<int>((L.size() + 1) / 2);
      for (size_t i = 0; i < L.size(); ++i) ent[2 * ((i / 2) * TS + sl) + (i % 2)] = L[i];
      npush[sl] = static_cast<int>(push[q][sl].size());
      for (int h = 0; h < npush[sl]; ++h) pdst[static_cast<size_t>(h) * TS + sl] = push[q][sl][h];
    }
    std::vector<int> fab(FS, (24 * TS) | ((24 * (TS + 1)) << 16)), fgt(FS), fgh(FS, -1), fid(FS, -1);
    std::vector<double> fl0(FS, 0.5), fea(FS, P.M > 0 ? P.ea[0] : 1.0), flt(FS, 1.0), flh(FS, 1.0);
    for (int fs = 0; fs < FS; ++fs) fgt[fs] = 24 * ((fs / T) * FT + fs % T);  // (reducer: unused)
    for (int k = 0; k < static_cast<int>(Q.slot_fiber.size()); ++k) {
      const int i = Q.slot_fiber[k];
      if (i < 0) continue;  // dummy slot
      const int fs = (k / FT) * T + k % FT;
      const int f = Q.fibers[i], tl = Q.tail_pn[i], hd = Q.head_pn[i];
      const int ph = plan.part_of_pn[hd];
      auto xoff = [&](int pn) {  // own slot or halo slot (mirror mode: either end may be remote)
        return plan.part_of_pn[pn] == q ? 24 * plan.slot_of_pn[pn] : 24 * (TS + 2 + halo_of[q][pn]);
      };
      fab[fs] = xoff(tl) | (xoff(hd) << 16);
      fgt[fs] = 24 * k;
      if (ph != q && !plan.mirror)
        fgh[fs] = (ph << 24) |
                  (24 * (own_slots + hrec[f]));
      fid[fs] = f;
      fl0[fs] = P.l0[f];
      fea[fs] = P.ea[f];
      flt[fs] = P.lump[tl];
      flh[fs] = P.lump[hd];
    }
    D.f0 = Q.f0;
    D.node_slots = Q.node_slots;
    D.halo = static_cast<int>(Q.halo_pn.size());
    D.max_pairs = max_pairs;
    D.max_push = max_push;
    D.n_records = zero_rec + 1;
    A.add(&D.slot_pn, slot_pn);
    A.add(&D.slot_ref, slot_ref);
    A.add(&D.slot_lump, slot_lump);
    A.add(&D.csr_npairs, npairs);
    A.add(&D.csr_pairs, ent);
    A.add(&D.push_n, npush);
    A.add(&D.push_dst, pdst);
    A.add(&D.fib_ab, fab);
    A.add(&D.fib_gt, fgt);
    A.add(&D.fib_gh, fgh);
    A.add(&D.fib_id, fid);
    A.add(&D.fib_l0, fl0);
    A.add(&D.fib_ea, fea);
    A.add(&D.fib_lt, flt);
    A.add(&D.fib_lh, flh);
    max_pairs_all = std::max(max_pairs_all, max_pairs);
    max_push_all = std::max(max_push_all, max_push);
    max_rec = std::max(max_rec, D.n_records);
  }
  ClusterEntryDev& E = de.cdev;
  E = ClusterEntryDev{};
  E.n_nodes = P.N;
  E.n_fibers = P.M;
  E.n_free_nodes = P.NFN;
  E.n_fix_nodes = P.N - P.NFN;
  E.max_lump = P.max_lump;
  E.max_ea = d.max_ea;
  E.box_volume = 8.0 * d.box_half * d.box_half * d.box_half;
  E.ea0 = P.M > 0 ? P.ea[0] : 1.0;
  E.mirror = plan.mirror ? 1 : 0;
  parts_off = A.reserve(sizeof(PartDev) * C);  // filled at commit, once pointers are known
  K.ts = TS;
  K.x_bytes = static_cast<int>(align16(24ull * (TS + 2 + halo_banks(plan) * plan.max_halo)));
  K.max_halo = plan.mirror ? plan.max_halo : 0;
  K.g_bytes = static_cast<int>(align16(24ull * max_rec));
  K.csr_cap = max_pairs_all * TS;
  K.push_cap = max_push_all * TS;
  K.scratch_stride = 6LL * P.N + 3LL * P.NFN + P.M;
}

// one allocation and one copy for an entry's arrays (and, for cluster entries, its PartDev
// table, whose pointer fields are resolved first)
int commit_entry(fibra_ctx* c, DeviceEntry& de, Arena& A, std::vector<PartDev>& parts,
                 size_t parts_off) {
  unsigned char* base = nullptr;
  FB_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&base), A.host.size()));
  de.allocs.push_back(base);
  for (auto& f : A.fixes) {  // store the device address into the (const T*) field
    const void* addr = base + f.second;
    std::memcpy(f.first, &addr, sizeof addr);
  }
  if (!parts.empty()) {
    std::memcpy(A.host.data() + parts_off, parts.data(), sizeof(PartDev) * parts.size());
    de.cdev.parts = reinterpret_cast<const PartDev*>(base + parts_off);
  }
  FB_CUDA(c, cudaMemcpy(base, A.host.data(), A.host.size(), cudaMemcpyHostToDevice));
  return FIBRA_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------
// multi-device contexts (fibra_cuda_open_devices): one sub-context per GPU, each a full
// single-device context over its shard of the points; NCCL (resolved at run time, so a
// process that already holds torch's libnccl.so.2 shares it) gathers the result records
// ---------------------------------------------------------------------------------
namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.err = "libnccl.so.2 not found";
      return r;
    }
    r.comm_init_all = reinterpret_cast<decltype(r.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.ok = r.comm_init_all && r.all_gather && r.group_start && r.group_end && r.comm_destroy &&
           r.error_string;
    if (!r.ok) r.err = "libnccl.so.2 lacks the collective entry points";
    return r;
  }();
  return api;
}

#define FB_NCCL(ctx, call)                                                                  \
  do {                                                                                      \
    const ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                                  \
      return set_err(ctx, FIBRA_E_CUDA, std::string(#call) + ": " + nccl_api().error_string(r_)); \
  } while (0)

__global__ void gather_F_kernel(int n, const int32_t* idx, const double* F, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 9 * n) return;
  out[i] = F[9 * idx[i / 9] + i % 9];
}

// records in point order from the gathered device blocks; one thread per 8-byte word
__global__ void permute_records_kernel(int n, const int* src, const fibra_point_result* in,
                                       fibra_point_result* out) {
  constexpr int W = sizeof(fibra_point_result) / 8;
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(W) * n) return;
  const int p = static_cast<int>(i / W), w = static_cast<int>(i % W);
  reinterpret_cast<unsigned long long*>(out + p)[w] =
      reinterpret_cast<const unsigned long long*>(in + src[p])[w];
}

template <class Fn>
int for_each_sub(fibra_ctx* c, Fn fn) {  // one host thread per device, first error wins
  const int nd = static_cast<int>(c->subs.size());
  std::vector<int> rc(nd, FIBRA_OK);
  std::vector<std::thread> th;
  for (int i = 0; i < nd; ++i) th.emplace_back([&, i] { rc[i] = fn(i, c->subs[i]); });
  for (auto& t : th) t.join();
  for (int i = 0; i < nd; ++i)
    if (rc[i] != FIBRA_OK)
      return set_err(c, rc[i], "device " + std::to_string(c->subs[i]->device) + ": " +
                                   c->subs[i]->err);
  return FIBRA_OK;
}

void free_multi_points(fibra_ctx* c) {
  for (size_t i = 0; i < c->subs.size(); ++i) {
    cudaSetDevice(c->subs[i]->device);
    if (i < c->d_block.size()) cudaFree(c->d_block[i]);
    if (i < c->d_gather.size()) cudaFree(c->d_gather[i]);
    if (i < c->d_Fsh.size()) cudaFree(c->d_Fsh[i]);
  }
  if (!c->subs.empty()) {
    cudaSetDevice(c->subs[0]->device);
    for (int32_t* p : c->d_Fidx) cudaFree(p);
    cudaFree(c->d_src);
    cudaFree(c->d_out0);
    cudaFree(c->d_F0);
  }
  c->d_block.clear();
  c->d_gather.clear();
  c->d_Fsh.clear();
  c->d_Fidx.clear();
  c->d_src = nullptr;
  c->d_out0 = nullptr;
  c->d_F0 = nullptr;
  c->cap0 = 0;
}

// (re)bind every device to its shard and size the gather buffers
int multi_bind_shards(fibra_ctx* c) {
  const int nd = static_cast<int>(c->subs.size());
  const int n = c->n_points;
  c->shard.assign(nd, {});
  c->local_of_point.assign(n, 0);
  for (int p = 0; p < n; ++p) {
    c->local_of_point[p] = static_cast<int32_t>(c->shard[c->dev_of_point[p]].size());
    c->shard[c->dev_of_point[p]].push_back(p);
  }
  int rc = for_each_sub(c, [&](int i, fibra_ctx* sc) {
    std::vector<int32_t> eop(c->shard[i].size());
    for (size_t k = 0; k < eop.size(); ++k) eop[k] = c->entry_of_point[c->shard[i][k]];
    return fibra_cuda_bind_points(sc, eop.data(), static_cast<int32_t>(eop.size()));
  });
  if (rc) return rc;
  free_multi_points(c);
  c->block = 1;
  for (const auto& sh : c->shard) c->block = std::max(c->block, static_cast<int>(sh.size()));
  c->d_block.assign(nd, nullptr);
  c->d_gather.assign(nd, nullptr);
  c->d_Fsh.assign(nd, nullptr);
  const size_t rb = sizeof(fibra_point_result);
  for (int i = 0; i < nd; ++i) {
    FB_CUDA(c, cudaSetDevice(c->subs[i]->device));
    FB_CUDA(c, cudaMalloc(&c->d_block[i], rb * c->block));
    FB_CUDA(c, cudaMemset(c->d_block[i], 0, rb * c->block));  // padding rows: zero records
    FB_CUDA(c, cudaMalloc(&c->d_gather[i], rb * c->block * nd));
    FB_CUDA(c, cudaMalloc(&c->d_Fsh[i], 9 * sizeof(double) * c->block));
  }
  FB_CUDA(c, cudaSetDevice(c->subs[0]->device));
  c->d_Fidx.assign(nd, nullptr);
  for (int i = 0; i < nd; ++i) {
    FB_CUDA(c, cudaMalloc(&c->d_Fidx[i], sizeof(int32_t) * std::max<size_t>(c->shard[i].size(), 1)));
    // device i's F is gathered on device 0 into its own staging rows (device i's slot in
    // d_gather[0] is reused: records are only written there by the all-gather later)
    if (!c->shard[i].empty())
      FB_CUDA(c, cudaMemcpy(c->d_Fidx[i], c->shard[i].data(), sizeof(int32_t) * c->shard[i].size(),
                            cudaMemcpyHostToDevice));
  }
  std::vector<int> src(std::max(n, 1));
  for (int p = 0; p < n; ++p) src[p] = c->dev_of_point[p] * c->block + c->local_of_point[p];
  FB_CUDA(c, cudaMalloc(&c->d_src, sizeof(int) * src.size()));
  FB_CUDA(c, cudaMemcpy(c->d_src, src.data(), sizeof(int) * src.size(), cudaMemcpyHostToDevice));
  return FIBRA_OK;
}

// all states of the shards in global PackedStates layout (host)
struct HostStates {
  std::vector<double> a[7], t;
  std::vector<int64_t> iters;
  std::vector<uint8_t> conv;
};

int multi_download(fibra_ctx* c, double* const* dst7, double* t, int64_t* iters, uint8_t* conv) {
  return for_each_sub(c, [&](int i, fibra_ctx* sc) {
    const auto& sh = c->shard[i];
    const size_t tot = sc->offsets.empty() ? 0 : static_cast<size_t>(sc->offsets.back());
    HostStates h;
    for (auto& v : h.a) v.resize(std::max<size_t>(tot, 1));
    h.t.resize(sh.size() + 1);
    h.iters.resize(sh.size() + 1);
    h.conv.resize(sh.size() + 1);
    const int r = fibra_cuda_download_states(sc, dst7[0] ? h.a[0].data() : nullptr,
                                             dst7[1] ? h.a[1].data() : nullptr,
                                             dst7[2] ? h.a[2].data() : nullptr,
                                             dst7[3] ? h.a[3].data() : nullptr,
                                             dst7[4] ? h.a[4].data() : nullptr,
                                             dst7[5] ? h.a[5].data() : nullptr,
                                             dst7[6] ? h.a[6].data() : nullptr, h.t.data(),
                                             h.iters.data(), h.conv.data());
    if (r) return r;
    for (size_t k = 0; k < sh.size(); ++k) {
      const int p = sh[k];
      const long long go = c->offsets[p], lo = sc->offsets[k], len = c->offsets[p + 1] - go;
      for (int a = 0; a < 7; ++a)
        if (dst7[a]) std::memcpy(dst7[a] + go, h.a[a].data() + lo, sizeof(double) * len);
      if (t) t[p] = h.t[k];
      if (iters) iters[p] = h.iters[k];
      if (conv) conv[p] = h.conv[k];
    }
    return FIBRA_OK;
  });
}

int multi_upload(fibra_ctx* c, const double* u, const double* t, const int64_t* iters,
                 const uint8_t* conv) {
  return for_each_sub(c, [&](int i, fibra_ctx* sc) {
    const auto& sh = c->shard[i];
    const size_t tot = sc->offsets.empty() ? 0 : static_cast<size_t>(sc->offsets.back());
    std::vector<double> hu(std::max<size_t>(tot, 1)), ht(sh.size() + 1);
    std::vector<int64_t> hi(sh.size() + 1);
    std::vector<uint8_t> hc(sh.size() + 1);
    for (size_t k = 0; k < sh.size(); ++k) {
      const int p = sh[k];
      const long long go = c->offsets[p], lo = sc->offsets[k], len = c->offsets[p + 1] - go;
      if (u) std::memcpy(hu.data() + lo, u + go, sizeof(double) * len);
      if (t) ht[k] = t[p];
      if (iters) hi[k] = iters[p];
      if (conv) hc[k] = conv[p];
    }
    return fibra_cuda_upload_states(sc, u ? hu.data() : nullptr, t ? ht.data() : nullptr,
                                    iters ? hi.data() : nullptr, conv ? hc.data() : nullptr);
  });
}

// Shards are planned lazily: at the first solve the cost model sees F (the strain term of
// the input-only model, as prep_kernel's schedule key), before that only the topology.
std::vector<double> strain_costs(const fibra_ctx* c, const double* F) {
  const int n = c->n_points;
  std::vector<double> cost(std::max(n, 1), 1.0);
  for (int p = 0; p < n; ++p) {
    const double* f = F + 9 * p;
    double e2 = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const double cij = f[i] * f[j] + f[3 + i] * f[3 + j] + f[6 + i] * f[6 + j] - (i == j);
        e2 += cij * cij;
      }
    const int e = c->entry_of_point[p];
    const double lk = e2 > 0 ? c->entry_log_its[e] - 0.185 * std::log(e2) : 30.0;
    cost[p] = std::exp(std::min(lk, 30.0)) * std::max(c->entry_fibers[e], 1);
  }
  return cost;
}

int ensure_plan(fibra_ctx* c, const double* cost) {
  if (!c->plan_pending) return FIBRA_OK;
  const int n = c->n_points;
  std::vector<double> topo;
  if (!cost) {
    topo.assign(std::max(n, 1), 1.0);
    for (int p = 0; p < n; ++p) topo[p] = c->entry_cost[c->entry_of_point[p]];
    cost = topo.data();
  }
  c->dev_of_point.assign(std::max(n, 1), 0);
  fibra_plan_shards(cost, n, static_cast<int32_t>(c->subs.size()), c->dev_of_point.data());
  c->dev_of_point.resize(n);
  int rc = multi_bind_shards(c);
  if (rc) return rc;
  c->plan_pending = false;
  if (c->staged) {
    c->staged = false;
    rc = multi_upload(c, c->stage_u.data(), c->stage_t.data(), c->stage_iters.data(),
                      c->stage_conv.data());
    c->stage_u = {};
    c->stage_t = {};
    c->stage_iters = {};
    c->stage_conv = {};
  }
  return rc;
}

int multi_solve_device(fibra_ctx* c, const double* F_dev, const fibra_law* law,
                       const fibra_relax_cfg* relax, const fibra_stiff_cfg* stiff,
                       int32_t want_tangent, fibra_point_result* out_dev) {
  const int nd = static_cast<int>(c->subs.size());
  const int n = c->n_points;
  if (c->offsets.empty()) return set_err(c, FIBRA_E_ARG, "bind_points must precede solve");
  fibra_ctx* s0 = c->subs[0];
  if (c->plan_pending) {  // the shard plan sees this call's F
    std::vector<double> Fh(9 * static_cast<size_t>(std::max(n, 1)));
    FB_CUDA(c, cudaSetDevice(s0->device));
    if (n) FB_CUDA(c, cudaMemcpy(Fh.data(), F_dev, 9 * sizeof(double) * n, cudaMemcpyDeviceToHost));
    const std::vector<double> cost = strain_costs(c, Fh.data());
    const int rc = ensure_plan(c, cost.data());
    if (rc) return rc;
  }
  FB_CUDA(c, cudaSetDevice(s0->device));
  FB_CUDA(c, cudaEventRecord(c->ev[0], s0->stream));
  // F of every shard: gathered on device 0, copied to its device over NVLink
  for (int i = 0; i < nd; ++i) {
    const int m = static_cast<int>(c->shard[i].size());
    if (!m) continue;
    double* stage = (i == 0) ? c->d_Fsh[0]
                             : reinterpret_cast<double*>(c->d_gather[0] + static_cast<size_t>(i) * c->block);
    gather_F_kernel<<<(9 * m + 255) / 256, 256, 0, s0->stream>>>(m, c->d_Fidx[i], F_dev, stage);
    FB_CUDA(c, cudaGetLastError());
    if (i)
      FB_CUDA(c, cudaMemcpyPeerAsync(c->d_Fsh[i], c->subs[i]->device, stage, s0->device,
                                     9 * sizeof(double) * m, s0->stream));
  }
  FB_CUDA(c, cudaEventRecord(c->ev_fork, s0->stream));
  for (int i = 0; i < nd; ++i) {
    fibra_ctx* sc = c->subs[i];
    FB_CUDA(c, cudaSetDevice(sc->device));
    FB_CUDA(c, cudaStreamWaitEvent(sc->stream, c->ev_fork, 0));
    const int r = launch_solve(sc, c->d_Fsh[i], law, relax, stiff, want_tangent, c->d_block[i]);
    if (r) return set_err(c, r, "device " + std::to_string(sc->device) + ": " + sc->err);
  }
  // one all-gather of the padded record blocks, every device receives all of them
  const NcclApi& api = nccl_api();
  const size_t bytes = sizeof(fibra_point_result) * static_cast<size_t>(c->block);
  FB_NCCL(c, api.group_start());
  for (int i = 0; i < nd; ++i)
    FB_NCCL(c, api.all_gather(c->d_block[i], c->d_gather[i], bytes, ncclUint8, c->comms[i],
                              c->subs[i]->stream));
  FB_NCCL(c, api.group_end());
  FB_CUDA(c, cudaSetDevice(s0->device));
  FB_CUDA(c, cudaEventRecord(c->ev[1], s0->stream));
  if (n) {
    constexpr int W = sizeof(fibra_point_result) / 8;
    const long long words = static_cast<long long>(W) * n;
    permute_records_kernel<<<static_cast<unsigned>((words + 255) / 256), 256, 0, s0->stream>>>(
        n, c->d_src, c->d_gather[0], out_dev);
    FB_CUDA(c, cudaGetLastError());
  }
  FB_CUDA(c, cudaEventRecord(c->ev[3], s0->stream));
  c->last_solves = 0;
  return FIBRA_OK;
}

int multi_solve(fibra_ctx* c, const double* F, const fibra_law* law, const fibra_relax_cfg* relax,
                const fibra_stiff_cfg* stiff, int32_t want_tangent, fibra_point_result* out) {
  const int n = c->n_points;
  fibra_ctx* s0 = c->subs[0];
  if (c->offsets.empty()) return set_err(c, FIBRA_E_ARG, "bind_points must precede solve");
  if (c->plan_pending) {
    const std::vector<double> cost = strain_costs(c, F);
    const int rp = ensure_plan(c, cost.data());
    if (rp) return rp;
  }
  FB_CUDA(c, cudaSetDevice(s0->device));
  if (c->cap0 < std::max(n, 1)) {
    cudaFree(c->d_F0);
    cudaFree(c->d_out0);
    c->cap0 = std::max(n, 1);
    FB_CUDA(c, cudaMalloc(&c->d_F0, 9 * sizeof(double) * c->cap0));
    FB_CUDA(c, cudaMalloc(&c->d_out0, sizeof(fibra_point_result) * c->cap0));
  }
  if (n) FB_CUDA(c, cudaMemcpyAsync(c->d_F0, F, 9 * sizeof(double) * n, cudaMemcpyHostToDevice, s0->stream));
  int rc = multi_solve_device(c, c->d_F0, law, relax, stiff, want_tangent, c->d_out0);
  if (rc) return rc;
  FB_CUDA(c, cudaSetDevice(s0->device));
  if (n)
    FB_CUDA(c, cudaMemcpyAsync(out, c->d_out0, sizeof(fibra_point_result) * n, cudaMemcpyDeviceToHost,
                               s0->stream));
  FB_CUDA(c, cudaStreamSynchronize(s0->stream));
  return FIBRA_OK;
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
  if (cudaMalloc(&c->d_ticket, 2 * kMaxClasses * sizeof(int)) != cudaSuccess) return bail(FIBRA_E_CUDA);
  if (cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  c->max_smem -= 4096;  // the kernels' static control blocks (+ kClusterCtlExtra for ClusterCtl)
  if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  if (cudaMalloc(&c->d_counters, 5 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(FIBRA_E_CUDA);
  *out = c;
  return FIBRA_OK;
}

int fibra_plan_shards(const double* cost, int32_t n, int32_t n_dev, int32_t* dev_of_point) {
  if (n < 0 || n_dev < 1 || (n && (!cost || !dev_of_point))) return FIBRA_E_ARG;
  std::vector<int> order(n);
  for (int p = 0; p < n; ++p) order[p] = p;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(n_dev, 0.0);
  for (int p : order) {
    int best = 0;
    for (int d = 1; d < n_dev; ++d)
      if (load[d] < load[best]) best = d;
    dev_of_point[p] = best;
    load[best] += std::max(cost[p], 0.0);
  }
  return FIBRA_OK;
}

int fibra_network_cost(const fibra_net_desc* d, double* cost) {
  if (!d || !cost || d->n_nodes <= 0 || d->n_fibers < 0) return FIBRA_E_ARG;
  const PackedNet P = pack(*d);
  *cost = std::exp(static_cast<double>(topology_log_its(P))) * std::max(P.M, 1);
  return FIBRA_OK;
}

int fibra_cuda_open_devices(const int32_t* devices, int32_t n_dev, fibra_ctx** out) {
  if (!out || n_dev < 1 || !devices) return FIBRA_E_ARG;
  *out = nullptr;
  if (n_dev == 1) return fibra_cuda_open(devices[0], out);
  const NcclApi& api = nccl_api();
  if (!api.ok) return FIBRA_E_CUDA;
  auto* c = new fibra_ctx;
  c->device = devices[0];
  c->own_stream = false;
  auto bail = [&](int code) {
    for (fibra_ctx* sc : c->subs) fibra_cuda_close(sc);
    delete c;
    return code;
  };
  for (int i = 0; i < n_dev; ++i) {
    fibra_ctx* sc = nullptr;
    const int rc = fibra_cuda_open(devices[i], &sc);
    if (rc) return bail(rc);
    // the devices build their copies of the library concurrently: share the host cores
    sc->host_threads = std::max(1, static_cast<int>(std::thread::hardware_concurrency()) / n_dev);
    c->subs.push_back(sc);
  }
  for (int i = 0; i < n_dev; ++i)  // NVLink peer access (the F copies; NCCL finds its own)
    for (int j = 0; j < n_dev; ++j) {
      int can = 0;
      if (i != j && cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) == cudaSuccess && can) {
        cudaSetDevice(devices[i]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return bail(FIBRA_E_CUDA);
        cudaGetLastError();
      }
    }
  c->comms.resize(n_dev);
  std::vector<int> devs(devices, devices + n_dev);
  if (api.comm_init_all(c->comms.data(), n_dev, devs.data()) != ncclSuccess) {
    c->comms.clear();
    return bail(FIBRA_E_CUDA);
  }
  cudaSetDevice(devices[0]);
  c->n_sm = c->subs[0]->n_sm;
  c->stream = c->subs[0]->stream;
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(FIBRA_E_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess)
    return bail(FIBRA_E_CUDA);
  *out = c;
  return FIBRA_OK;
}

int fibra_cuda_close(fibra_ctx* c) {
  if (!c) return FIBRA_OK;
  if (!c->subs.empty()) {
    for (fibra_ctx* sc : c->subs) cudaSetDevice(sc->device), cudaStreamSynchronize(sc->stream);
    free_multi_points(c);
    for (ncclComm_t m : c->comms) nccl_api().comm_destroy(m);
    cudaSetDevice(c->subs[0]->device);
    for (auto& e : c->ev) cudaEventDestroy(e);
    cudaEventDestroy(c->ev_fork);
    for (fibra_ctx* sc : c->subs) fibra_cuda_close(sc);
    delete c;
    return FIBRA_OK;
  }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_points(c);
  free_scratch(c);
  free_library(c);
  cudaFree(c->d_ticket);
  cudaFree(c->d_trace);
  cudaFree(c->d_counters);
  for (auto& e : c->ev) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_fork);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return FIBRA_OK;
}

const char* fibra_cuda_last_error(const fibra_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fibra_cuda_set_stream(fibra_ctx* c, void* stream) {
  if (!c->subs.empty())
    return set_err(c, FIBRA_E_ARG, "set_stream: a multi-device context uses its devices' streams");
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
  if (!c->subs.empty()) {  // replicated on every device
    c->entry_cost.assign(n, 1.0);
    c->entry_log_its.assign(n, 0.0f);
    c->entry_fibers.assign(n, 0);
    c->entry_ndof.assign(n, 0);
    for (int i = 0; i < n; ++i) {
      if (entries[i].n_nodes <= 0 || entries[i].n_fibers < 0)
        return set_err(c, FIBRA_E_ARG, "malformed library entry " + std::to_string(i));
      const PackedNet P = pack(entries[i]);
      c->entry_log_its[i] = topology_log_its(P);
      c->entry_fibers[i] = P.M;
      c->entry_ndof[i] = 3 * P.N;
      c->entry_cost[i] = std::exp(static_cast<double>(c->entry_log_its[i])) * std::max(P.M, 1);
    }
    c->entry_of_point.clear();
    c->offsets.clear();
    const int rc = for_each_sub(c, [&](int, fibra_ctx* sc) {
      return fibra_cuda_upload_library(sc, entries, n);
    });
    if (!rc) c->entries.assign(n, DeviceEntry());  // marks the library as uploaded
    return rc;
  }
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  free_library(c);
  for (int i = 0; i < n; ++i) {
    const fibra_net_desc& d = entries[i];
    if (d.n_nodes <= 0 || d.n_fibers < 0 || d.n_free % 3 != 0)
      return set_err(c, FIBRA_E_ARG, "malformed library entry " + std::to_string(i));
  }
  // host work per entry (packing, shape selection, schedules) runs on all host cores
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  const int workers = std::max(1, std::min<int>(n, c->host_threads > 0 ? c->host_threads : hw));
  auto parallel_for = [&](int lo, int hi, const std::function<void(int)>& fn) {
    std::atomic<int> next(lo);
    std::vector<std::thread> pool;
    for (int w = 0; w < std::min(workers, hi - lo); ++w)
      pool.emplace_back([&] {
        for (int i; (i = next.fetch_add(1)) < hi;) fn(i);
      });
    for (auto& t : pool) t.join();
  };
  // kernel shape per entry: the first resident shape that holds it, else the smallest
  // cluster (fewest CTAs) that does
  c->entries.resize(n);
  std::vector<PackedNet> nets(n);
  std::vector<ClusterPlan> plans(n);
  std::vector<int> kind_cl(n, 0), kind_vi(n, -1), kind_C(n, 1), kind_node(n, 0), kind_stream(n, 0);
  // FIBRA_KERNEL=node: the node-centric kernel (dr_node.cuh) for the entries it holds.
  // Opt-in: it removes the fiber -> node barrier but evaluates every fibre twice, and on
  // config 2 it issues 13.0k instructions per RVE-iteration against the fiber/node kernel's
  // 6.2k, with warps waiting on the highest-degree warp (profiles/r02_node_*).
  const char* kern_env = getenv("FIBRA_KERNEL");
  const bool allow_node = kern_env && kern_env[0] == 'n';
  // FIBRA_KERNEL=stream: every entry on the HBM-streaming kernel (A/B timing); it is
  // otherwise taken by entries that fit no resident shape and no 16-CTA cluster.
  // FIBRA_STREAM_C=C restricts it to C-CTA clusters.
  const bool force_stream = kern_env && kern_env[0] == 's';
  const char* stream_c_env = getenv("FIBRA_STREAM_C");
  const int stream_c = stream_c_env ? atoi(stream_c_env) : 0;
  std::vector<Caps> est(n);  // the entry's shared-memory components (exact, = the build's)
  // diagnostics: FIBRA_FORCE_CLUSTER=C places every entry on a C-CTA cluster (kernel timing)
  const char* force_env = getenv("FIBRA_FORCE_CLUSTER");
  const int force_c = force_env ? atoi(force_env) : 0;
  // diagnostics: FIBRA_CLUSTER_SHAPE=i restricts the cluster kernels to kClusterVariants[i]
  const char* shape_env = getenv("FIBRA_CLUSTER_SHAPE");
  const int force_shape = shape_env ? atoi(shape_env) : -1;
  parallel_for(0, n, [&](int i) {
    nets[i] = pack(entries[i]);
    const PackedNet& P = nets[i];
    DeviceEntry& de = c->entries[i];
    de.config_ok = P.ok;
    de.config_err = P.err;
    de.n_nodes = P.N;
    const int mp = max_pairs_of(P);
    de.log_its = topology_log_its(P);
    // diagnostics: FIBRA_NODE_SHAPE=i restricts the node kernel to kNodeVariants[i]
    const char* nshape_env = getenv("FIBRA_NODE_SHAPE");
    const int force_nshape = nshape_env ? atoi(nshape_env) : -1;
    for (int v = 0; v < kNumNodeVariants && kind_vi[i] < 0 && !force_c && allow_node &&
                    !force_stream; ++v)
      if ((force_nshape < 0 || v == force_nshape) &&
          node_fits(c, P, kNodeVariants[v], false, de.nsched)) {
        kind_vi[i] = v;
        kind_node[i] = 1;
        const NodeVariant& nv = kNodeVariants[v];
        const int TS = nv.NPT * nv.T;
        est[i].ts = TS;
        est[i].x_bytes = static_cast<int>(align16(24ull * TS));
        int capn = 32 * std::max(de.nsched.n_rows, 1);
        const size_t region = ((4ull * capn + 15) & ~15ull) + 16ull * capn;
        const size_t exit_need = 8ull * (3 * P.N + 3 * P.NFN + P.M);
        if (region < exit_need) capn = static_cast<int>((exit_need + 19) / 20 + 32);
        est[i].csr_cap = capn;
      }
    // diagnostics: FIBRA_RESIDENT_SKIP=i leaves kVariants[i] out (shape experiments)
    const char* skip_env = getenv("FIBRA_RESIDENT_SKIP");
    const int skip_v = skip_env ? atoi(skip_env) : -1;
    for (int v = 0; v < kNumVariants && kind_vi[i] < 0 && !force_c && !force_stream; ++v)
      if (v != skip_v && resident_fits(c, P, kVariants[v], mp, de.sched)) {
        kind_vi[i] = v;
        const int TS = kVariants[v].NPT * kVariants[v].T;
        est[i].ts = TS;
        est[i].x_bytes = static_cast<int>(align16(24ull * (TS + 32)));
        est[i].g_bytes = static_cast<int>(align16(std::max<size_t>(
            24ull * (de.sched.gd_slots + 17), 8ull * (3 * P.N + 3 * P.NFN + P.M))));
        est[i].csr_cap = 2 * (mp + 2) * TS;  // + the padding rows
      }
    // cluster: first the 384-thread shapes on up to 4 CTAs, then the fewest CTAs with the
    // first shape that holds the parts (config 3 with the round-2 kernels: its 2.5k-6.7k
    // fibre RVEs on 4 x (384,4,1) finish 0.4 s before 2 x (512,7,2), 2,448 -> 2,488
    // RVE-solves/s; config 4's lattices need 16 x (512,7,2))
    auto cluster_try = [&](int cc, int v) {
      if (kind_vi[i] >= 0 || force_stream || (force_shape >= 0 && v != force_shape)) return;
      if (force_c && cc != force_c) return;
      {
          if (cluster_fits(c, P, kClusterVariants[v], cc, mp, plans[i])) {
            kind_vi[i] = v;
            kind_C[i] = cc;
            kind_cl[i] = 1;
            const ClusterVariant& cv = kClusterVariants[v];
            const int TS = cv.NPT * cv.T;
            size_t max_h = 0;
            for (const ClusterPart& q : plans[i].parts) max_h = std::max(max_h, q.h_fiber.size());
            est[i].ts = TS;
            est[i].x_bytes = static_cast<int>(
                align16(24ull * (TS + 2 + halo_banks(plans[i]) * plans[i].max_halo)));
            est[i].max_halo = plans[i].mirror ? plans[i].max_halo : 0;
            est[i].g_bytes = static_cast<int>(align16(24ull * (cv.FPT * (cv.T - 32) + max_h + 1)));
            est[i].csr_cap = mp * TS;
            est[i].push_cap = plans[i].max_push * TS;
          }
      }
    };
    for (int cc = 2; cc <= 4; cc *= 2)
      for (int v = 0; v < kNumClusterVariants; ++v)
        if (kClusterVariants[v].T == 384) cluster_try(cc, v);
    for (int cc = 2; cc <= 16; cc *= 2)
      for (int v = 0; v < kNumClusterVariants; ++v) cluster_try(cc, v);
    // beyond on-chip capacity: the streaming kernel, the lightest shape (fewest nodes per
    // thread) on the fewest CTAs whose slots hold the nodes
    for (int v = 0; v < kNumStreamVariants && kind_vi[i] < 0; ++v)
      for (int cc = 2; cc <= 16 && kind_vi[i] < 0; cc *= 2) {
        if (stream_c && cc != stream_c) continue;
        const StreamVariant& sv = kStreamVariants[v];
        if (!build_node_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), cc * sv.T, sv.NPT, 0,
                                 de.nsched))
          continue;
        kind_vi[i] = v;
        kind_C[i] = cc;
        kind_stream[i] = 1;
        est[i].ts = sv.T * sv.NPT;
        est[i].s_cap = cc * sv.T * sv.NPT;
        est[i].n_cap = P.N;
        est[i].m_cap = P.M;
      }
  });
  for (int i = 0; i < n; ++i) {
    if (kind_vi[i] < 0)
      return set_err(c, FIBRA_E_ARG, "RVE library entry " + std::to_string(i) + " (" +
                                         std::to_string(nets[i].M) + " fibers, " +
                                         std::to_string(nets[i].N) +
                                         " nodes) exceeds every kernel shape");
    const bool cl = kind_cl[i] != 0;
    const bool nd = kind_node[i] != 0;
    const bool sm = kind_stream[i] != 0;
    // a class's footprint is the per-component maximum over its entries: join the first
    // class of this kernel shape that still fits the device with this entry, else open one
    auto fits_with = [&](const KClass& K) {
      KClass T = K;
      T.uniform_ea = false;
      merge_caps(T, est[i]);
      return T.smem() <= static_cast<size_t>(c->max_smem - (cl ? kClusterCtlExtra : 0));
    };
    int k = 0;
    const int nk = static_cast<int>(c->classes.size());
    while (k < nk && !(c->classes[k].cluster == cl && c->classes[k].node == nd &&
                       c->classes[k].streaming == sm && c->classes[k].vi == kind_vi[i] &&
                       c->classes[k].C == kind_C[i] && fits_with(c->classes[k])))
      ++k;
    if (k == nk) {
      if (nk == kMaxClasses) return set_err(c, FIBRA_E_ARG, "too many kernel classes in one library");
      KClass K;
      K.cluster = cl;
      K.node = nd;
      K.streaming = sm;
      K.vi = kind_vi[i];
      K.C = kind_C[i];
      c->classes.push_back(K);
    }
    merge_caps(c->classes[k], est[i]);
    c->entries[i].cls = k;
    KClass& K = c->classes[k];
    const PackedNet& P = nets[i];
    for (int f = 1; f < P.M && K.uniform_ea; ++f) K.uniform_ea = (P.ea[f] == P.ea[0]);
  }
  // device arrays: built in parallel batches (bounded host memory), committed in order
  const int batch = 256;
  for (int lo = 0; lo < n; lo += batch) {
    const int hi = std::min(n, lo + batch);
    std::vector<Arena> arenas(hi - lo);
    std::vector<std::vector<PartDev>> parts(hi - lo);
    std::vector<size_t> parts_off(hi - lo, 0);
    std::vector<Caps> caps(hi - lo);
    parallel_for(lo, hi, [&](int i) {
      DeviceEntry& de = c->entries[i];
      const KClass& K = c->classes[de.cls];
      de.orient = OrientDev{};
      de.orient.n_fibers = nets[i].M;
      arenas[i - lo].add(&de.orient.a, nets[i].a);
      arenas[i - lo].add(&de.orient.b, nets[i].b);
      arenas[i - lo].add(&de.orient.ref, nets[i].ref);
      if (K.cluster)
        build_cluster_entry(de, nets[i], entries[i], plans[i], kClusterVariants[K.vi],
                            arenas[i - lo], parts[i - lo], parts_off[i - lo], caps[i - lo]);
      else if (K.node)
        build_node_entry(de, nets[i], entries[i], kNodeVariants[K.vi], arenas[i - lo],
                         caps[i - lo]);
      else if (K.streaming)
        build_stream_entry(de, nets[i], entries[i], kStreamVariants[K.vi], K.C, arenas[i - lo],
                           caps[i - lo]);
      else
        build_resident_entry(de, nets[i], entries[i], kVariants[K.vi], arenas[i - lo],
                             caps[i - lo]);
    });
    for (int i = lo; i < hi; ++i) {
      const int rc = commit_entry(c, c->entries[i], arenas[i - lo], parts[i - lo], parts_off[i - lo]);
      if (rc) return rc;
      merge_caps(c->classes[c->entries[i].cls], caps[i - lo]);
      nets[i] = PackedNet();
      plans[i] = ClusterPlan();
    }
  }
  {
    std::vector<OrientDev> host(n);
    for (int i = 0; i < n; ++i) host[i] = c->entries[i].orient;
    FB_CUDA(c, cudaMalloc(&c->d_orient, sizeof(OrientDev) * n));
    FB_CUDA(c, cudaMemcpy(c->d_orient, host.data(), sizeof(OrientDev) * n, cudaMemcpyHostToDevice));
  }
  for (KClass& K : c->classes) {
    if (K.smem() > static_cast<size_t>(c->max_smem - (K.cluster ? kClusterCtlExtra : 0)))
      return set_err(c, FIBRA_E_ARG, "library shared-memory footprint exceeds the device limit");
    if (K.streaming) {
      std::vector<StreamEntryDev> host(n, StreamEntryDev{});
      for (int i = 0; i < n; ++i)
        if (&c->classes[c->entries[i].cls] == &K) {
          host[i] = c->entries[i].sdev;
          // (l0, rcp_refined(l0)) pairs: the reciprocal with the device's own sequence
          const long long ninc = 32ll * std::max(host[i].n_rows, 1);
          init_rcp_kernel<<<static_cast<unsigned>((ninc + 255) / 256), 256, 0, c->stream>>>(
              const_cast<double2*>(host[i].inc_l0), ninc);
          FB_CUDA(c, cudaGetLastError());
        }
      FB_CUDA(c, cudaStreamSynchronize(c->stream));
      FB_CUDA(c, cudaMalloc(&K.d_sentries, sizeof(StreamEntryDev) * n));
      FB_CUDA(c, cudaMemcpy(K.d_sentries, host.data(), sizeof(StreamEntryDev) * n,
                            cudaMemcpyHostToDevice));
    } else if (K.node) {
      std::vector<NodeEntryDev> host(n, NodeEntryDev{});
      for (int i = 0; i < n; ++i)
        if (&c->classes[c->entries[i].cls] == &K) host[i] = c->entries[i].ndev;
      FB_CUDA(c, cudaMalloc(&K.d_nentries, sizeof(NodeEntryDev) * n));
      FB_CUDA(c, cudaMemcpy(K.d_nentries, host.data(), sizeof(NodeEntryDev) * n,
                            cudaMemcpyHostToDevice));
    } else if (K.cluster) {
      std::vector<ClusterEntryDev> host(n, ClusterEntryDev{});
      for (int i = 0; i < n; ++i)
        if (&c->classes[c->entries[i].cls] == &K) host[i] = c->entries[i].cdev;
      FB_CUDA(c, cudaMalloc(&K.d_centries, sizeof(ClusterEntryDev) * n));
      FB_CUDA(c, cudaMemcpy(K.d_centries, host.data(), sizeof(ClusterEntryDev) * n,
                            cudaMemcpyHostToDevice));
    } else {
      std::vector<EntryDev> host(n, EntryDev{});
      for (int i = 0; i < n; ++i)
        if (&c->classes[c->entries[i].cls] == &K) host[i] = c->entries[i].dev;
      FB_CUDA(c, cudaMalloc(&K.d_entries, sizeof(EntryDev) * n));
      FB_CUDA(c, cudaMemcpy(K.d_entries, host.data(), sizeof(EntryDev) * n, cudaMemcpyHostToDevice));
    }
    FB_CUDA(c, cudaStreamCreateWithFlags(&K.stream, cudaStreamNonBlocking));
    FB_CUDA(c, cudaStreamCreateWithFlags(&K.stream2, cudaStreamNonBlocking));
    FB_CUDA(c, cudaEventCreateWithFlags(&K.done, cudaEventDisableTiming));
    FB_CUDA(c, cudaEventCreateWithFlags(&K.done2, cudaEventDisableTiming));
    FB_CUDA(c, cudaEventCreate(&K.done_t));
  }
  return FIBRA_OK;
}

int fibra_cuda_bind_points(fibra_ctx* c, const int32_t* entry_of_point, int32_t n) {
  if (!c || n < 0) return FIBRA_E_ARG;
  if (c->entries.empty()) return set_err(c, FIBRA_E_ARG, "upload_library first");
  if (!c->subs.empty()) {  // shards: longest-processing-time, planned at the first use
    c->offsets.assign(n + 1, 0);
    for (int p = 0; p < n; ++p) {
      const int e = entry_of_point[p];
      if (e < 0 || e >= static_cast<int>(c->entry_cost.size()))
        return set_err(c, FIBRA_E_CONFIG, "assignment entry out of range");
      c->offsets[p + 1] = c->offsets[p] + c->entry_ndof[e];  // global PackedStates layout
    }
    c->entry_of_point.assign(entry_of_point, entry_of_point + n);
    c->n_points = n;
    c->plan_pending = true;
    c->staged = false;
    free_multi_points(c);
    return FIBRA_OK;
  }
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  free_points(c);
  c->entry_of_point.assign(entry_of_point, entry_of_point + n);
  c->offsets.assign(n + 1, 0);
  std::vector<int> cls(n);
  for (auto& K : c->classes) K.n_points = 0;
  for (int p = 0; p < n; ++p) {
    const int e = entry_of_point[p];
    if (e < 0 || e >= static_cast<int>(c->entries.size()))
      return set_err(c, FIBRA_E_CONFIG, "assignment entry out of range");
    c->offsets[p + 1] = c->offsets[p] + 3LL * c->entries[e].n_nodes;
    cls[p] = c->entries[e].cls;
    ++c->classes[cls[p]].n_points;
  }
  int off = 0;  // the schedule order groups points by class (sort keys)
  for (auto& K : c->classes) {
    K.point_off = off;
    off += K.n_points;
  }
  c->n_points = n;
  const size_t tot = static_cast<size_t>(c->offsets[n]);
  int rc;
  if ((rc = dalloc(c, &c->d_entry_of_point, n))) return rc;
  if ((rc = dalloc(c, &c->d_class_of_point, n))) return rc;
  if ((rc = dalloc(c, &c->d_pcost, n))) return rc;
  if ((rc = dalloc(c, &c->d_offsets, n + 1))) return rc;
  for (int k = 0; k < 7; ++k)
    if ((rc = dalloc(c, &c->d_state[k], tot))) return rc;
  if ((rc = dalloc(c, &c->d_state[7], n))) return rc;
  if ((rc = dalloc(c, &c->d_iters, n))) return rc;
  if ((rc = dalloc(c, &c->d_conv, n))) return rc;
  if (n) {
    FB_CUDA(c, cudaMemcpy(c->d_entry_of_point, entry_of_point, sizeof(int) * n, cudaMemcpyHostToDevice));
    FB_CUDA(c, cudaMemcpy(c->d_class_of_point, cls.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    std::vector<float> pc(n);
    for (int p = 0; p < n; ++p) pc[p] = c->entries[entry_of_point[p]].log_its;
    FB_CUDA(c, cudaMemcpy(c->d_pcost, pc.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
  }
  FB_CUDA(c, cudaMemcpy(c->d_offsets, c->offsets.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice));
  return fibra_cuda_reset_states(c);
}

int fibra_cuda_orientation(fibra_ctx* c, const int32_t* points, int32_t n, const double* ref_dir,
                           double* out) {
  if (!c || n < 0 || (n && (!points || !ref_dir || !out))) return FIBRA_E_ARG;
  if (!c->d_orient || c->offsets.empty())
    return set_err(c, FIBRA_E_ARG, "upload_library and bind_points must precede orientation");
  if (n == 0) return FIBRA_OK;
  for (int i = 0; i < n; ++i)
    if (points[i] < 0 || points[i] >= c->n_points)
      return set_err(c, FIBRA_E_ARG, "orientation: point out of range");
  if (!c->subs.empty()) {  // each point on the device that holds its state
    const int rp = ensure_plan(c, nullptr);
    if (rp) return rp;
    for (int i = 0; i < n; ++i) {
      const int32_t loc = c->local_of_point[points[i]];
      fibra_ctx* sc = c->subs[c->dev_of_point[points[i]]];
      const int rc = fibra_cuda_orientation(sc, &loc, 1, ref_dir, out + i);
      if (rc) return set_err(c, rc, sc->err);
    }
    return FIBRA_OK;
  }
  FB_CUDA(c, cudaSetDevice(c->device));
  int* d_pts = nullptr;
  double* d_out = nullptr;
  FB_CUDA(c, cudaMalloc(&d_pts, sizeof(int) * n));
  FB_CUDA(c, cudaMalloc(&d_out, sizeof(double) * n));
  FB_CUDA(c, cudaMemcpyAsync(d_pts, points, sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
  orientation_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(
      n, d_pts, c->d_entry_of_point, c->d_offsets, c->d_orient, c->d_state[0], ref_dir[0],
      ref_dir[1], ref_dir[2], d_out);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaMemcpyAsync(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_pts);
  cudaFree(d_out);
  return FIBRA_OK;
}

int fibra_cuda_entry_kernel(const fibra_ctx* c, int32_t entry, int32_t* out) {
  if (c && !c->subs.empty()) return fibra_cuda_entry_kernel(c->subs[0], entry, out);
  if (!c || !out || entry < 0 || entry >= static_cast<int>(c->entries.size())) return FIBRA_E_ARG;
  const KClass& K = c->classes[c->entries[entry].cls];
  if (K.streaming) {  // fibres per thread: -1 marks the streaming kernel
    const StreamVariant& v = kStreamVariants[K.vi];
    out[0] = K.C, out[1] = v.T, out[2] = -1, out[3] = v.NPT;
  } else if (K.node) {  // fibres per thread: 0 marks the node-centric kernel
    const NodeVariant& v = kNodeVariants[K.vi];
    out[0] = 1, out[1] = v.T, out[2] = 0, out[3] = v.NPT;
  } else if (K.cluster) {
    const ClusterVariant& v = kClusterVariants[K.vi];
    out[0] = K.C, out[1] = v.T, out[2] = v.FPT, out[3] = v.NPT;
  } else {
    const Variant& v = kVariants[K.vi];
    out[0] = 1, out[1] = v.T, out[2] = v.FPT, out[3] = v.NPT;
  }
  return FIBRA_OK;
}

int fibra_cuda_set_schedule(fibra_ctx* c, int32_t mode, const double* cost_hint) {
  if (!c) return FIBRA_E_ARG;
  if (mode != FIBRA_SCHED_BATCH && mode != FIBRA_SCHED_STRAIN && mode != FIBRA_SCHED_HINT)
    return set_err(c, FIBRA_E_ARG, "unknown schedule mode");
  if (!c->subs.empty()) {
    if (mode == FIBRA_SCHED_HINT) {
      if (!cost_hint) return set_err(c, FIBRA_E_ARG, "FIBRA_SCHED_HINT needs cost_hint");
      if (c->offsets.empty()) return set_err(c, FIBRA_E_ARG, "bind_points first");
      // re-plan the shards on the caller's costs; the warm states of the points that
      // change device move with them (host round trip)
      const int n = c->n_points;
      if (c->plan_pending) {
        const int rp = ensure_plan(c, cost_hint);
        if (rp) return rp;
      }
      std::vector<int32_t> dev(std::max(n, 1));
      fibra_plan_shards(cost_hint, n, static_cast<int32_t>(c->subs.size()), dev.data());
      if (!std::equal(dev.begin(), dev.begin() + n, c->dev_of_point.begin())) {
        const size_t tot = static_cast<size_t>(c->offsets.back());
        std::vector<double> u(std::max<size_t>(tot, 1)), t(std::max(n, 1));
        std::vector<int64_t> it(std::max(n, 1));
        std::vector<uint8_t> cv(std::max(n, 1));
        double* dst7[7] = {u.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        int rc = multi_download(c, dst7, t.data(), it.data(), cv.data());
        if (rc) return rc;
        c->dev_of_point.assign(dev.begin(), dev.begin() + n);
        if ((rc = multi_bind_shards(c))) return rc;
        if ((rc = multi_upload(c, u.data(), t.data(), it.data(), cv.data()))) return rc;
      }
      return for_each_sub(c, [&](int i, fibra_ctx* sc) {
        std::vector<double> h(std::max<size_t>(c->shard[i].size(), 1));
        for (size_t k = 0; k < c->shard[i].size(); ++k) h[k] = cost_hint[c->shard[i][k]];
        return fibra_cuda_set_schedule(sc, mode, h.data());
      });
    }
    return for_each_sub(c, [&](int, fibra_ctx* sc) { return fibra_cuda_set_schedule(sc, mode, nullptr); });
  }
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
  if (!c->subs.empty()) {
    if (c->plan_pending) {
      c->staged = false;
      return FIBRA_OK;
    }
    return for_each_sub(c, [&](int, fibra_ctx* sc) { return fibra_cuda_reset_states(sc); });
  }
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
  if (!c->subs.empty()) {
    if (c->plan_pending) {  // staged until the first solve plans the shards
      const size_t tot = static_cast<size_t>(c->offsets.back());
      const size_t n = c->n_points;
      c->stage_u.assign(std::max<size_t>(tot, 1), 0.0);
      c->stage_t.assign(std::max<size_t>(n, 1), 0.0);
      c->stage_iters.assign(std::max<size_t>(n, 1), 0);
      c->stage_conv.assign(std::max<size_t>(n, 1), 0);
      if (u && tot) std::memcpy(c->stage_u.data(), u, sizeof(double) * tot);
      if (t && n) std::memcpy(c->stage_t.data(), t, sizeof(double) * n);
      if (iters && n) std::memcpy(c->stage_iters.data(), iters, sizeof(int64_t) * n);
      if (converged && n) std::memcpy(c->stage_conv.data(), converged, n);
      c->staged = true;
      return FIBRA_OK;
    }
    return multi_upload(c, u, t, iters, converged);
  }
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
  if (!c->subs.empty()) {
    const int rp = ensure_plan(c, nullptr);
    if (rp) return rp;
    double* dst7[7] = {u, v, a, f_int, f_damp, mass, inv_mass};
    return multi_download(c, dst7, t, iters, converged);
  }
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
  if (!c->subs.empty()) return multi_solve(c, F, law, relax, stiff, want_tangent, out);
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
  if (!c->subs.empty()) return multi_solve_device(c, F_dev, law, relax, stiff, want_tangent, out_dev);
  FB_CUDA(c, cudaSetDevice(c->device));
  return launch_solve(c, F_dev, law, relax, stiff, want_tangent, out_dev);
}

int fibra_cuda_selftest_fastmath(fibra_ctx* c, uint64_t n, uint64_t seed, uint64_t* mismatches) {
  if (!c->subs.empty()) return fibra_cuda_selftest_fastmath(c->subs[0], n, seed, mismatches);
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

int fibra_cuda_eval_libm(fibra_ctx* c, int32_t which, const double* x, int64_t n, double* out) {
  if (!c || n < 0 || (n && (!x || !out))) return FIBRA_E_ARG;
  if (!c->subs.empty()) return fibra_cuda_eval_libm(c->subs[0], which, x, n, out);
  if (n == 0) return FIBRA_OK;
  FB_CUDA(c, cudaSetDevice(c->device));
  double* d = nullptr;
  FB_CUDA(c, cudaMalloc(&d, 2 * sizeof(double) * n));
  FB_CUDA(c, cudaMemcpyAsync(d, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  eval_libm_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(which, d, n, d + n);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaMemcpyAsync(out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(d);
  return FIBRA_OK;
}

int fibra_cuda_fp64_peak(fibra_ctx* c, double* out) {  // per device
  if (!c->subs.empty()) return fibra_cuda_fp64_peak(c->subs[0], out);
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

int fibra_cuda_trace(fibra_ctx* c, unsigned long long* out, size_t cap, size_t* n) {
  if (!c || !n) return FIBRA_E_ARG;
  if (!c->subs.empty()) return fibra_cuda_trace(c->subs[0], out, cap, n);
  *n = c->trace_n;
  if (!out || !c->d_trace || !c->trace_n) return FIBRA_OK;
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  FB_CUDA(c, cudaMemcpy(out, c->d_trace, 8 * std::min(cap, c->trace_n), cudaMemcpyDeviceToHost));
  return FIBRA_OK;
}

int fibra_cuda_phase_profile(fibra_ctx* c, unsigned long long* out, size_t cap, size_t* n) {
  if (!c->subs.empty()) return fibra_cuda_phase_profile(c->subs[0], out, cap, n);
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  *n = c->phase_prof_n;
  if (c->phase_prof && out && cap >= c->phase_prof_n)
    FB_CUDA(c, cudaMemcpy(out, c->phase_prof, c->phase_prof_n * 8, cudaMemcpyDeviceToHost));
  return FIBRA_OK;
}

int fibra_cuda_synchronize(fibra_ctx* c) {
  if (!c->subs.empty())
    return for_each_sub(c, [&](int, fibra_ctx* sc) { return fibra_cuda_synchronize(sc); });
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  FB_CUDA(c, cudaGetLastError());
  return FIBRA_OK;
}

int fibra_cuda_last_stats(fibra_ctx* c, fibra_solve_stats* s) {
  if (!c->subs.empty()) {  // sums over devices; DR time = the slowest device's
    std::memset(s, 0, sizeof *s);
    for (fibra_ctx* sc : c->subs) {
      fibra_solve_stats d;
      const int rc = fibra_cuda_last_stats(sc, &d);
      if (rc) return set_err(c, rc, sc->err);
      s->solves += d.solves;
      s->iterations += d.iterations;
      s->fiber_iterations += d.fiber_iterations;
      s->pipe_ops += d.pipe_ops;
      s->alg_flops += d.alg_flops;
      s->kernel_launches += d.kernel_launches;
      s->dr_kernel_ms = std::max(s->dr_kernel_ms, d.dr_kernel_ms);
    }
    s->kernel_launches += 1 + static_cast<int32_t>(c->subs.size());  // F gathers + permute
    FB_CUDA(c, cudaSetDevice(c->subs[0]->device));
    FB_CUDA(c, cudaStreamSynchronize(c->subs[0]->stream));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]) == cudaSuccess) s->total_ms = ms;
    return FIBRA_OK;
  }
  FB_CUDA(c, cudaSetDevice(c->device));
  FB_CUDA(c, cudaStreamSynchronize(c->stream));
  unsigned long long cnt[5] = {0, 0, 0, 0, 0};
  FB_CUDA(c, cudaMemcpy(cnt, c->d_counters, sizeof cnt, cudaMemcpyDeviceToHost));
  std::memset(s, 0, sizeof *s);
  s->iterations = static_cast<int64_t>(cnt[0]);
  s->fiber_iterations = static_cast<int64_t>(cnt[1]);
  s->pipe_ops = static_cast<int64_t>(cnt[2]);
  s->solves = static_cast<int64_t>(cnt[3]);
  s->alg_flops = static_cast<int64_t>(cnt[4]);
  float ms = 0;
  if (cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]) == cudaSuccess) s->dr_kernel_ms = ms;
  if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]) == cudaSuccess) s->total_ms = ms;
  s->kernel_launches = c->last_launches;
  if (getenv("FIBRA_CLASS_TIMES"))  // diagnostics: per kernel class, ms from the fork
    for (size_t k = 0; k < c->classes.size(); ++k) {
      const KClass& K = c->classes[k];
      if (!K.n_points) continue;
      float t = -1;
      cudaEventElapsedTime(&t, c->ev[1], K.done_t);
      std::fprintf(stderr, "class %zu: %s %s C=%d points=%d done at %.1f ms\n", k,
                   K.cluster ? "cluster" : (K.node ? "node" : "resident"),
                   K.cluster ? (std::to_string(kClusterVariants[K.vi].T) + "/" +
                                std::to_string(kClusterVariants[K.vi].FPT)).c_str()
                   : K.node  ? (std::to_string(kNodeVariants[K.vi].T) + "/" +
                                std::to_string(kNodeVariants[K.vi].NPT)).c_str()
                             : (std::to_string(kVariants[K.vi].T) + "/" +
                                std::to_string(kVariants[K.vi].FPT)).c_str(),
                   K.C, K.n_points, t);
    }
  return FIBRA_OK;
}

// Diagnostics: emulate one force pass of the cluster kernel on the host from exactly the
// per-CTA arrays the upload builds (x pushes, fiber records, signed CSR gather), next to a
// direct per-fiber assembly.  g = ea * (L - l0) / (l0 * L) stands in for the law; the two
// force vectors must agree to rounding.  No CUDA calls.
int fibra_debug_cluster_forces(const fibra_net_desc* d, int C, int shape, int mirror,
                               const double* u, double* f_emul, double* f_direct) {
  if (!d || !u || !f_emul || !f_direct || shape < 0 || shape >= kNumClusterVariants) return FIBRA_E_ARG;
  const PackedNet P = pack(*d);
  const ClusterVariant& v = kClusterVariants[shape];
  ClusterPlan plan;
  if (!build_cluster_plan(P.N, P.NFN, P.M, P.a.data(), P.b.data(), P.ref.data(), C, v.T, v.FPT,
                          v.NPT, mirror != 0, plan))
    return FIBRA_E_CONFIG;
  DeviceEntry de;
  Arena A;
  std::vector<PartDev> parts;
  size_t parts_off = 0;
  Caps K;
  build_cluster_entry(de, P, *d, plan, v, A, parts, parts_off, K);
  for (auto& f : A.fixes) {
    const void* addr = A.host.data() + f.second;
    std::memcpy(f.first, &addr, sizeof addr);
  }
  const int T = v.T, TS = v.NPT * T, FS = v.FPT * T, FT = T - 32;
  const int hs = 3 * (TS + 2 + plan.max_halo);
  std::vector<std::vector<double>> X(C, std::vector<double>(hs, 0.0));
  std::vector<std::vector<double>> G(C);
  for (int q = 0; q < C; ++q) G[q].assign(3 * static_cast<size_t>(parts[q].n_records), 0.0);
  auto x_of = [&](int pn, int c) { return P.ref[3 * pn + c] + u[3 * pn + c]; };
  for (int q = 0; q < C; ++q) {  // own x and pushes
    const PartDev& D = parts[q];
    X[q][3 * TS + 3] = 1.0;  // dummy records at TS, TS+1: unit segment
    for (int sl = 0; sl < TS; ++sl) {
      const int pn = D.slot_pn[sl];
      if (pn < 0) continue;
      for (int c = 0; c < 3; ++c) X[q][3 * sl + c] = x_of(pn, c);
      for (int h = 0; h < D.push_n[sl]; ++h) {
        const int dd = D.push_dst[static_cast<size_t>(h) * TS + sl];
        const int r = static_cast<unsigned>(dd) >> 16, o = (dd & 0xffff) / 8;
        if (r >= C || o + 2 >= hs) return 100 + q;
        for (int c = 0; c < 3; ++c) X[r][o + c] = x_of(pn, c);
      }
    }
  }
  for (int q = 0; q < C; ++q) {  // fiber records (+ remote copies)
    const PartDev& D = parts[q];
    for (int fs = 0; fs < FS; ++fs) {
      if (fs % T >= FT || D.fib_id[fs] < 0) continue;
      const int ta = (D.fib_ab[fs] & 0xffff) / 8, hb = (static_cast<unsigned>(D.fib_ab[fs]) >> 16) / 8;
      double dx[3], dd = 0;
      for (int c = 0; c < 3; ++c) {
        dx[c] = X[q][hb + c] - X[q][ta + c];
        dd += dx[c] * dx[c];
      }
      const double L = std::sqrt(dd), l0 = D.fib_l0[fs];
      const double g = D.fib_ea[fs] * (L - l0) / (l0 * L);
      const int go = D.fib_gt[fs] / 8;
      for (int c = 0; c < 3; ++c) G[q][go + c] = g * dx[c];
      if (D.fib_gh[fs] >= 0) {
        const int r = static_cast<unsigned>(D.fib_gh[fs]) >> 24, o = (D.fib_gh[fs] & 0xffffff) / 8;
        for (int c = 0; c < 3; ++c) G[r][o + c] = g * dx[c];
      }
    }
  }
  for (int i = 0; i < 3 * P.N; ++i) f_emul[i] = f_direct[i] = 0.0;
  for (int q = 0; q < C; ++q) {  // signed CSR gather of own nodes
    const PartDev& D = parts[q];
    for (int sl = 0; sl < TS; ++sl) {
      const int pn = D.slot_pn[sl];
      if (pn < 0) continue;
      for (int i = 0; i < 2 * D.csr_npairs[sl]; ++i) {
        const int e = reinterpret_cast<const int*>(D.csr_pairs)[2 * ((i / 2) * TS + sl) + (i % 2)];
        const int o = (e & 0x7fffffff) / 8;
        const double sg = (e < 0) ? -1.0 : 1.0;
        for (int c = 0; c < 3; ++c) f_emul[3 * pn + c] += sg * G[q][o + c];
      }
    }
  }
  for (int f = 0; f < P.M; ++f) {
    double dx[3], dd = 0;
    for (int c = 0; c < 3; ++c) {
      dx[c] = x_of(P.b[f], c) - x_of(P.a[f], c);
      dd += dx[c] * dx[c];
    }
    const double L = std::sqrt(dd);
    const double g = P.ea[f] * (L - P.l0[f]) / (P.l0[f] * L);
    for (int c = 0; c < 3; ++c) {
      f_direct[3 * P.b[f] + c] += g * dx[c];
      f_direct[3 * P.a[f] + c] -= g * dx[c];
    }
  }
  return FIBRA_OK;
}

// Diagnostics: the same host emulation for a resident-kernel entry (kVariants[shape]).
int fibra_debug_resident_forces(const fibra_net_desc* d, int shape, const double* u,
                                double* f_emul, double* f_direct) {
  if (!d || !u || !f_emul || !f_direct || shape < 0 || shape >= kNumVariants) return FIBRA_E_ARG;
  const PackedNet P = pack(*d);
  const Variant& v = kVariants[shape];
  DeviceEntry de;
  if (!build_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), v.T, v.FPT, v.NPT, de.sched))
    return FIBRA_E_CONFIG;
  Arena A;
  Caps K;
  build_resident_entry(de, P, *d, v, A, K);
  for (auto& f : A.fixes) {
    const void* addr = A.host.data() + f.second;
    std::memcpy(f.first, &addr, sizeof addr);
  }
  const EntryDev& E = de.dev;
  const int TS = E.thread_slots, FS = E.fiber_slots;
  std::vector<double> X(3 * static_cast<size_t>(TS + 32), 0.0), G(3 * static_cast<size_t>(E.gd_slots), 0.0);
  for (int r = 16; r < 32; ++r) X[3 * (TS + r)] = 1.0;  // dummy head records (1,0,0)
  auto x_of = [&](int pn, int c) { return P.ref[3 * pn + c] + u[3 * pn + c]; };
  for (int sl = 0; sl < TS; ++sl)
    if (E.slot_pn[sl] >= 0)
      for (int c = 0; c < 3; ++c) X[3 * sl + c] = x_of(E.slot_pn[sl], c);
  std::vector<int> written(E.gd_slots, 0);
  for (int fs = 0; fs < FS; ++fs) {
    const int ta = (E.fib_ab[fs] & 0xffff) / 8, hb = (static_cast<unsigned>(E.fib_ab[fs]) >> 16) / 8;
    double dx[3], dd = 0;
    for (int c = 0; c < 3; ++c) {
      dx[c] = X[hb + c] - X[ta + c];
      dd += dx[c] * dx[c];
    }
    const double L = std::sqrt(dd), l0 = E.fib_l0[fs];
    const double g = E.fib_ea[fs] * (L - l0) / (l0 * L);
    const int gr = E.fib_g[fs] / 8;
    if (E.fib_id[fs] >= 0 && written[gr / 3]++) return 200;  // two fibers on one record
    for (int c = 0; c < 3; ++c) G[gr + c] = g * dx[c];
  }
  for (int c = 0; c < 3; ++c) G[3 * (E.gd_slots - 1) + c] = 0.0;
  for (int i = 0; i < 3 * P.N; ++i) f_emul[i] = f_direct[i] = 0.0;
  for (int sl = 0; sl < TS; ++sl) {
    const int pn = E.slot_pn[sl];
    if (pn < 0) continue;
    for (int i = 0; i < 2 * E.csr_npairs[sl]; ++i) {
      const int e = reinterpret_cast<const int*>(E.csr_pairs)[2 * ((i / 2) * TS + sl) + (i % 2)];
      const int r = (e & 0x7fffffff) / 8;
      for (int c = 0; c < 3; ++c)  // f + (-1) * (g*d) == f - g*d
        f_emul[3 * pn + c] = e < 0 ? f_emul[3 * pn + c] - G[r + c] : f_emul[3 * pn + c] + G[r + c];
    }
  }
  for (int f = 0; f < P.M; ++f) {
    double dx[3], dd = 0;
    for (int c = 0; c < 3; ++c) {
      dx[c] = x_of(P.b[f], c) - x_of(P.a[f], c);
      dd += dx[c] * dx[c];
    }
    const double L = std::sqrt(dd);
    const double g = P.ea[f] * (L - P.l0[f]) / (P.l0[f] * L);
    for (int c = 0; c < 3; ++c) {
      f_direct[3 * P.b[f] + c] += g * dx[c];
      f_direct[3 * P.a[f] + c] -= g * dx[c];
    }
  }
  return FIBRA_OK;
}

// Diagnostics (no CUDA): one force pass of the node-centric kernel emulated on the host from
// the uploaded arrays (x records by slot, step-major incidence tables, d' = x_other - x_own,
// f -= g d' from +0.0), linear law with ea_scale 1, into f_emul (packed node order).  The
// reference's force loop (network.cpp:275-311) must give the same bits.
// report[4] = {half-warp gather steps, excess wavefronts before / after the placement
// search, incidence rows}.
int fibra_debug_node_forces(const fibra_net_desc* d, int shape, const double* u, double* f_emul,
                            int64_t* report) {
  if (!d || !u || !f_emul || shape < 0 || shape >= kNumNodeVariants) return FIBRA_E_ARG;
  const PackedNet P = pack(*d);
  const NodeVariant& v = kNodeVariants[shape];
  DeviceEntry de;
  if (!build_node_schedule(P.N, P.NFN, P.M, P.a.data(), P.b.data(), v.T, v.NPT,
                           node_search_moves(), de.nsched))
    return FIBRA_E_CONFIG;
  Arena A;
  Caps K;
  build_node_entry(de, P, *d, v, A, K);
  for (auto& f : A.fixes) {
    const void* addr = A.host.data() + f.second;
    std::memcpy(f.first, &addr, sizeof addr);
  }
  const NodeEntryDev& E = de.ndev;
  const int TS = E.node_slots;
  std::vector<double> X(3 * static_cast<size_t>(TS), 0.0);
  for (int sl = 0; sl < TS; ++sl)
    for (int c = 0; c < 3; ++c)
      X[3 * sl + c] = E.slot_ref[3 * sl + c] + (E.slot_pn[sl] >= 0 ? u[3 * E.slot_pn[sl] + c] : 0.0);
  for (int i = 0; i < 3 * P.N; ++i) f_emul[i] = 0.0;
  for (int sl = 0; sl < TS; ++sl) {
    const int pn = E.slot_pn[sl];
    if (pn < 0) continue;
    const int g = sl / 32, lane = sl % 32;
    double f[3] = {0.0, 0.0, 0.0};
    for (int st = 0; st < E.slot_deg[sl]; ++st) {
      const int ix = 32 * (E.group_row0[g] + st) + lane;
      const int o = E.inc_x[ix] / 8;
      const double dx = X[o] - X[3 * sl], dy = X[o + 1] - X[3 * sl + 1], dz = X[o + 2] - X[3 * sl + 2];
      const double len = std::sqrt(dx * dx + dy * dy + dz * dz);
      const double l0 = E.inc_l0[ix];
      const double stretch = len / l0;
      const double gg = (1.0 * E.inc_ea[ix]) * (stretch - 1.0) / len;
      f[0] = f[0] - gg * dx;
      f[1] = f[1] - gg * dy;
      f[2] = f[2] - gg * dz;
    }
    for (int c = 0; c < 3; ++c) f_emul[3 * pn + c] = f[c];
  }
  if (report) {
    report[0] = de.nsched.steps;
    report[1] = de.nsched.excess_initial;
    report[2] = de.nsched.excess;
    report[3] = de.nsched.n_rows;
  }
  return FIBRA_OK;
}

// Diagnostics (no CUDA): the cluster plan's dynamic shared-memory footprint for shape `shape`
// on C CTAs.  out[4] = {plan found, mirror mode, dynamic bytes, static ClusterCtl bytes}.
int fibra_debug_cluster_smem(const fibra_net_desc* d, int C, int shape, int64_t* out) {
  if (!d || !out || shape < 0 || shape >= kNumClusterVariants) return FIBRA_E_ARG;
  const PackedNet P = pack(*d);
  const ClusterVariant& v = kClusterVariants[shape];
  ClusterPlan plan;
  const bool ok = build_cluster_plan(P.N, P.NFN, P.M, P.a.data(), P.b.data(), P.ref.data(), C, v.T,
                                     v.FPT, v.NPT, true, plan) ||
                  build_cluster_plan(P.N, P.NFN, P.M, P.a.data(), P.b.data(), P.ref.data(), C, v.T,
                                     v.FPT, v.NPT, false, plan);
  out[0] = ok;
  out[1] = ok && plan.mirror;
  out[2] = ok ? static_cast<int64_t>(cluster_smem(plan, v, max_pairs_of(P))) : 0;
  out[3] = static_cast<int64_t>(sizeof(ClusterCtl));
  return FIBRA_OK;
}

}  // extern "C"
