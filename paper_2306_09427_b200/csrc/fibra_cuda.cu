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
#include <cstring>
#include <string>
#include <vector>

#include "dr_kernel.cuh"
#include "fibra_cuda.h"
#include "tensor.cuh"

namespace fibra_b200 {

struct PrepOut {
  double R[9];
  double U[6];
  double h;
  int status;
  int pad;
};

__global__ void prep_kernel(int n, const double* __restrict__ F, int want_tangent,
                            double fd_rel_step, PrepOut* prep, double* solve_F, int* solve_skip,
                            int* base_flag) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double f[9];
  for (int i = 0; i < 9; ++i) f[i] = F[9 * p + i];
  PrepOut o = {};
  base_flag[p] = 0;
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

__global__ void post_kernel(int n, const double* __restrict__ F, int want_tangent,
                            const PrepOut* __restrict__ prep, const SolveOut* __restrict__ out,
                            fibra_point_result* res) {
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
  double probe_pk2[36];
  if (!status && want_tangent) {
    for (int q = 0; q < 6 && !status; ++q) {
      const SolveOut& o = out[n + 6 * p + q];
      if (o.status) {
        status = FIBRA_E_PROBE_FAILED;
        failed_probe = q;
      } else {
        its += o.iterations;
        for (int i = 0; i < 6; ++i) probe_pk2[6 * q + i] = o.pk2[i];
      }
    }
    if (!status) {
      if (!material_stiffness_from_probes(pr.U, b.pk2, probe_pk2, pr.h, r.material_a))
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
  rotate_stress(pr.R, b.sigma_u, r.sigma);
  for (int i = 0; i < 6; ++i) r.pk2[i] = b.pk2[i];
  r.stress_asymmetry = b.asym;
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
  int T, FPT, NPT, LAW;
  KernelFn fn;
};

#define FB_V(T, F, N, L) {T, F, N, L, &dr_persistent_kernel<T, F, N, L>}
static const Variant kVariants[] = {
    FB_V(512, 1, 1, 0), FB_V(512, 2, 1, 0), FB_V(512, 4, 1, 0), FB_V(512, 4, 2, 0),
    FB_V(512, 8, 2, 0), FB_V(512, 8, 4, 0), FB_V(256, 4, 2, 0), FB_V(256, 2, 1, 0),
    FB_V(512, 1, 1, 1), FB_V(512, 2, 1, 1), FB_V(512, 4, 1, 1), FB_V(512, 4, 2, 1),
    FB_V(512, 8, 2, 1), FB_V(512, 8, 4, 1), FB_V(256, 4, 2, 1), FB_V(256, 2, 1, 1),
};
#undef FB_V

struct DeviceEntry {
  EntryDev dev;
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
  int nmax = 0, mmax = 0;
  // points
  int n_points = 0;
  std::vector<int32_t> entry_of_point;
  std::vector<long long> offsets;
  int* d_entry_of_point = nullptr;
  long long* d_offsets = nullptr;
  double* d_state[8] = {};  // u v a f_int f_damp mass inv_mass t
  long long* d_iters = nullptr;
  unsigned char* d_conv = nullptr;
  // per-call scratch
  int cap_points = 0;
  double* d_F = nullptr;
  double* d_solveF = nullptr;
  int* d_skip = nullptr;
  PrepOut* d_prep = nullptr;
  SolveOut* d_out = nullptr;
  int* d_flag = nullptr;
  fibra_point_result* d_res = nullptr;
  double* h_F = nullptr;                 // pinned staging
  fibra_point_result* h_res = nullptr;   // pinned staging
  int* d_ticket = nullptr;
  unsigned long long* d_counters = nullptr;
  cudaEvent_t ev[4] = {};
  int last_solves = 0;
  int last_launches = 0;
};

namespace {

int set_err(fibra_ctx* c, int code, const std::string& what) {
  if (c) c->err = what;
  return code;
}

#define FB_CUDA(ctx, call)                                                           \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
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
  cudaFree(c->d_res);
  cudaFreeHost(c->h_F);
  cudaFreeHost(c->h_res);
  c->d_F = c->d_solveF = nullptr;
  c->d_skip = c->d_flag = nullptr;
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
  c->nmax = c->mmax = 0;
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
  if ((rc = dalloc(c, &c->d_res, n))) return rc;
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_F), 9 * sizeof(double) * n));
  FB_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_res), sizeof(fibra_point_result) * n));
  c->cap_points = n;
  return FIBRA_OK;
}

size_t smem_bytes(int nmax, int mmax) {
  const size_t bsize = std::max<size_t>(3 * static_cast<size_t>(mmax), 6 * static_cast<size_t>(nmax) + mmax);
  return sizeof(double) * (3 * static_cast<size_t>(nmax) + bsize + nmax) +
         sizeof(int) * (nmax + 1 + 2 * static_cast<size_t>(mmax));
}

const Variant* pick_variant(int nmax, int mmax, int law) {
  // smallest register footprint that covers the largest entry; prefer T=512
  const Variant* best = nullptr;
  for (const Variant& v : kVariants) {
    if (v.LAW != law || v.T != 512) continue;
    if (v.FPT * v.T < mmax || v.NPT * v.T < nmax) continue;
    if (!best || v.FPT + 3 * v.NPT < best->FPT + 3 * best->NPT) best = &v;
  }
  return best;
}

int launch_solve(fibra_ctx* c, const double* dF, const fibra_law* law,
                 const fibra_relax_cfg* rc, const fibra_stiff_cfg* sc, int want_tangent,
                 fibra_point_result* dres) {
  const int n = c->n_points;
  if (!c->d_entries || n == 0 && c->entry_of_point.empty())
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
  const Variant* v = pick_variant(c->nmax, c->mmax, law->kind);
  if (!v) return set_err(c, FIBRA_E_ARG, "RVE too large for the resident kernel variants");
  const size_t smem = smem_bytes(c->nmax, c->mmax);
  FB_CUDA(c, cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  int per_sm = 0;
  FB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v->fn, v->T, smem));
  if (per_sm < 1) return set_err(c, FIBRA_E_ARG, "DR kernel does not fit on an SM");
  const int n_solves = want_tangent ? 7 * n : n;
  const int grid = std::min(n_solves, per_sm * c->n_sm);

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
  P.ticket = c->d_ticket;
  P.counters = c->d_counters;
  P.n_points = n;
  P.n_solves = n_solves;
  P.nmax = c->nmax;
  P.mmax = c->mmax;
  P.reuse_warm = sc ? sc->reuse_warm : 1;
  P.law_buckling_off = law->buckling_off;
  P.ea_scale = law->ea_scale;
  P.nonlinearity = law->nonlinearity;
  P.damping = rc->damping;
  P.tolerance = rc->tolerance;
  P.dt_safety = rc->dt_safety;
  P.density_scale = rc->density_scale;
  P.max_iterations = rc->max_iterations;

  cudaStream_t st = c->stream;
  FB_CUDA(c, cudaEventRecord(c->ev[0], st));
  FB_CUDA(c, cudaMemsetAsync(c->d_ticket, 0, sizeof(int), st));
  FB_CUDA(c, cudaMemsetAsync(c->d_counters, 0, 4 * sizeof(unsigned long long), st));
  const int tb = 128;
  prep_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, sc ? sc->fd_rel_step : 1e-5,
                                                c->d_prep, c->d_solveF, c->d_skip, c->d_flag);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[1], st));
  v->fn<<<grid, v->T, smem, st>>>(P);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[2], st));
  post_kernel<<<(n + tb - 1) / tb, tb, 0, st>>>(n, dF, want_tangent, c->d_prep, c->d_out, dres);
  FB_CUDA(c, cudaGetLastError());
  FB_CUDA(c, cudaEventRecord(c->ev[3], st));
  c->last_solves = n_solves;
  c->last_launches = 3;
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
  if (cudaMalloc(&c->d_ticket, sizeof(int)) != cudaSuccess) return bail(FIBRA_E_CUDA);
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
  c->entries.resize(n);
  std::vector<EntryDev> host(n);
  for (int i = 0; i < n; ++i) {
    const fibra_net_desc& d = entries[i];
    DeviceEntry& de = c->entries[i];
    const int N = d.n_nodes, M = d.n_fibers;
    if (N <= 0 || N >= 65536 || M < 0 || d.n_free % 3 != 0)
      return set_err(c, FIBRA_E_ARG, "unsupported network size in library entry " + std::to_string(i));
    // packed-node views of the reference layout (free-first packing, network.cpp:120-143)
    std::vector<int> node_of_pn(N);
    for (int node = 0; node < N; ++node) node_of_pn[d.packed_of_dof[3 * node] / 3] = node;
    std::vector<double> lump(N);
    double max_lump = 0;
    for (int pn = 0; pn < N; ++pn) {
      lump[pn] = d.node_lump[node_of_pn[pn]];
      if (!(lump[pn] > 0) && de.config_ok) {  // setup_mass relax.cpp:29-31
        de.config_ok = false;
        de.config_err = "node " + std::to_string(node_of_pn[pn]) +
                        " has no incident fibers (singular mass)";
      }
      max_lump = (max_lump < lump[pn]) ? lump[pn] : max_lump;
    }
    std::vector<int> ab(M);
    std::vector<double> ea(M);
    std::vector<int> off(N + 1, 0), ent(2 * static_cast<size_t>(M));
    for (int f = 0; f < M; ++f) {
      const int a = d.fiber_packed_dofs[6 * f] / 3, b = d.fiber_packed_dofs[6 * f + 3] / 3;
      ab[f] = a | (b << 16);
      ea[f] = d.fiber_area[f] * d.fiber_modulus[f];  // FiberNetwork::fiber_ea
      ++off[a + 1];
      ++off[b + 1];
    }
    for (int pn = 0; pn < N; ++pn) off[pn + 1] += off[pn];
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (int f = 0; f < M; ++f) {  // ascending fiber id within every node's list
      const int a = ab[f] & 0xffff, b = ab[f] >> 16;
      ent[fill[a]++] = (f << 1) | 1;
      ent[fill[b]++] = (f << 1);
    }
    EntryDev& E = host[i];
    E.n_nodes = N;
    E.n_fibers = M;
    E.n_free_nodes = d.n_free / 3;
    E.max_lump = max_lump;
    E.max_ea = d.max_ea;
    E.box_volume = 8.0 * d.box_half * d.box_half * d.box_half;  // RveBox::volume
    auto up = [&](auto** dst, const auto* src, size_t count) -> int {
      using Tp = std::remove_const_t<std::remove_pointer_t<decltype(src)>>;
      Tp* p = nullptr;
      FB_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(Tp)));
      de.allocs.push_back(p);
      if (count) FB_CUDA(c, cudaMemcpy(p, src, count * sizeof(Tp), cudaMemcpyHostToDevice));
      *dst = p;
      return FIBRA_OK;
    };
    int rc;
    if ((rc = up(&E.ref, d.packed_ref, 3 * static_cast<size_t>(N)))) return rc;
    if ((rc = up(&E.lump, lump.data(), N))) return rc;
    if ((rc = up(&E.fiber_ab, ab.data(), M))) return rc;
    if ((rc = up(&E.l0, d.rest_length, M))) return rc;
    if ((rc = up(&E.ea, ea.data(), M))) return rc;
    if ((rc = up(&E.csr_off, off.data(), N + 1))) return rc;
    if ((rc = up(&E.csr_ent, ent.data(), 2 * static_cast<size_t>(M)))) return rc;
    de.dev = E;
    c->nmax = std::max(c->nmax, N);
    c->mmax = std::max(c->mmax, M);
  }
  c->nmax = (c->nmax + 1) & ~1;  // keep double/int regions aligned
  c->mmax = (c->mmax + 1) & ~1;
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

int fibra_cuda_fp64_peak(fibra_ctx* c, double* out) {
  FB_CUDA(c, cudaSetDevice(c->device));
  double* sink = nullptr;
  FB_CUDA(c, cudaMalloc(&sink, 1024 * sizeof(double)));
  const int iters = 1 << 16, blocks = 4 * c->n_sm, threads = 256;
  fp64_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink, 64, 1e-9);  // warm-up
  FB_CUDA(c, cudaEventRecord(c->ev[0], c->stream));
  fp64_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink, iters, 1e-9);
  FB_CUDA(c, cudaEventRecord(c->ev[3], c->stream));
  FB_CUDA(c, cudaEventSynchronize(c->ev[3]));
  float ms = 0;
  FB_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]));
  cudaFree(sink);
  *out = 8.0 * iters * static_cast<double>(blocks) * threads / (ms * 1e-3);
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
