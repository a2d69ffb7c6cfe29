// assembly.cu -- macro assembly of the homogenized responses on the device.
//
// Restates fibra::assemble (/root/reference/proj/src/macrofem.cpp:104-187) with b_matrix
// (:41-60) and mandel_b (:64-86): per linear tet, f_e = V B^T sigma and
// K_e = V B^T C B + geometric part, scattered into the free residual and the free x free
// stiffness exactly as Eigen::SparseMatrix::setFromTriplets folds the triplets (first value,
// then acc = acc + next in triplet order = element order; compressed column-major, rows
// sorted).  Results are bit-identical to the reference (compiled with --fmad=false like the
// rest of the library; every sum keeps the reference's operation order).
//
// B200 layout.  The sparsity pattern is topology only, so it is planned once per mesh on the
// host (assembly_create) and the per-Newton-iteration work is two HBM-streaming kernels:
//   asm_element_kernel: 12 threads per tet (thread r owns row/column r of K_e), 8 tets per
//     96-thread CTA; the response records (sigma + Mandel C, 42 doubles, any record stride,
//     e.g. the fibra_point_result array a device solve left in HBM) are staged in shared
//     memory, K_e is written as 16 contiguous 3x3 node blocks [b][a][ax][bx] (column node major) so the gather
//     reads 72 contiguous bytes per (node pair, element).
//   asm_pair_kernel: three threads (one per row axis) per (row node A, column node B) pair
//     with a free dof on both sides; each walks the elements shared by A and B in ascending
//     order and writes its (up to) 3 folded values straight into their compressed-column
//     slots.
//   asm_residual_kernel: one thread per node, the f_e entries of its elements in element
//     order, then residual -= f_ext (:185).
// Errors follow the reference's order: the first element (in element order) with a
// non-finite stress (:122-125, FIBRA_E_ASM_STRESS) or an inverted tet (:128-132,
// FIBRA_E_KINEMATICS), then a non-finite residual (:186-187, FIBRA_E_ASM_RESIDUAL).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "fibra_cuda.h"

namespace {

constexpr double kSqrt2 = 1.4142135623730951;  // macrofem.cpp:62
constexpr int kTetsPerCta = 8;
constexpr int kElemThreads = 12 * kTetsPerCta;
constexpr int kKeStride = 146;  // padded K_e staging: elements of one warp on distinct banks

__device__ __forceinline__ double cof3(const double* m, int i, int j) {
  // Eigen InverseImpl.h cofactor_3x3<i, j>
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[3 * i1 + j1] * m[3 * i2 + j2] - m[3 * i1 + j2] * m[3 * i2 + j1];
}

// b_matrix (macrofem.cpp:41-60); returns det (the caller tests det > 0)
__device__ __forceinline__ double tet_geom(const double* x, double grad[12], double* vol) {
  double jac[9];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) jac[3 * r + c] = x[3 * (c + 1) + r] - x[r];
  // Eigen determinant_impl<3> (row-0 expansion)
  const double det = jac[0] * (jac[4] * jac[8] - jac[5] * jac[7]) -
                     jac[1] * (jac[3] * jac[8] - jac[5] * jac[6]) +
                     jac[2] * (jac[3] * jac[7] - jac[4] * jac[6]);
  // Eigen compute_inverse<3>: its own det from the column-0 cofactors
  const double c0 = cof3(jac, 0, 0), c1 = cof3(jac, 1, 0), c2 = cof3(jac, 2, 0);
  const double idet = 1.0 / ((c0 * jac[0] + c1 * jac[3]) + c2 * jac[6]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) grad[3 * (a + 1) + k] = cof3(jac, k, a) * idet;
#pragma unroll
  for (int k = 0; k < 3; ++k) grad[k] = -grad[3 + k] - grad[6 + k] - grad[9 + k];
  *vol = det / 6.0;
  return det;
}

// column c = 3 node + ax of mandel_b (macrofem.cpp:64-86), accumulated onto zeros; shear
// rows (23, 13, 12) = pairs (1,2) (0,2) (0,1)
__device__ __forceinline__ void b_column(const double* grad, int c, double bc[6]) {
  const int node = c / 3, ax = c % 3;
  const double g0 = grad[3 * node], g1 = grad[3 * node + 1], g2 = grad[3 * node + 2];
  const double gax = ax == 0 ? g0 : (ax == 1 ? g1 : g2);
  bc[0] = ax == 0 ? 0.0 + gax : 0.0;
  bc[1] = ax == 1 ? 0.0 + gax : 0.0;
  bc[2] = ax == 2 ? 0.0 + gax : 0.0;
  // sh 0 (1,2): ax 1 -> 0.5 g2, ax 2 -> 0.5 g1; sh 1 (0,2): ax 0 -> 0.5 g2, ax 2 -> 0.5 g0;
  // sh 2 (0,1): ax 0 -> 0.5 g1, ax 1 -> 0.5 g0  (v = 0 + 0.5 g, else v = 0)
  const double v0 = ax == 1 ? 0.0 + 0.5 * g2 : (ax == 2 ? 0.0 + 0.5 * g1 : 0.0);
  const double v1 = ax == 0 ? 0.0 + 0.5 * g2 : (ax == 2 ? 0.0 + 0.5 * g0 : 0.0);
  const double v2 = ax == 0 ? 0.0 + 0.5 * g1 : (ax == 1 ? 0.0 + 0.5 * g0 : 0.0);
  bc[3] = 0.0 + kSqrt2 * v0;
  bc[4] = 0.0 + kSqrt2 * v1;
  bc[5] = 0.0 + kSqrt2 * v2;
}

// The three structurally non-zero rows of column c = 3 node + ax of mandel_b, ascending:
// ax 0 -> rows 0, 4, 5; ax 1 -> 1, 3, 5; ax 2 -> 2, 3, 4 (same values as b_column).
// Skipping the structural zeros is exact: a sum that starts at +0.0 never becomes -0.0, so
// adding a +-0 product leaves it unchanged -- provided the other factor is finite (an inf
// or NaN would turn the product into NaN); callers fall back to the dense loops otherwise.
__device__ __forceinline__ double sel6(const double v[6], int i) {  // no local-memory indexing
  return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : i == 3 ? v[3] : i == 4 ? v[4] : v[5];
}

__device__ __forceinline__ void b_column_sparse(const double* grad, int c, int rows[3],
                                                double v[3]) {
  const int node = c / 3, ax = c % 3;
  const double g0 = grad[3 * node], g1 = grad[3 * node + 1], g2 = grad[3 * node + 2];
  if (ax == 0) {
    rows[0] = 0, rows[1] = 4, rows[2] = 5;
    v[0] = 0.0 + g0, v[1] = 0.0 + kSqrt2 * (0.0 + 0.5 * g2), v[2] = 0.0 + kSqrt2 * (0.0 + 0.5 * g1);
  } else if (ax == 1) {
    rows[0] = 1, rows[1] = 3, rows[2] = 5;
    v[0] = 0.0 + g1, v[1] = 0.0 + kSqrt2 * (0.0 + 0.5 * g2), v[2] = 0.0 + kSqrt2 * (0.0 + 0.5 * g0);
  } else {
    rows[0] = 2, rows[1] = 3, rows[2] = 4;
    v[0] = 0.0 + g2, v[1] = 0.0 + kSqrt2 * (0.0 + 0.5 * g1), v[2] = 0.0 + kSqrt2 * (0.0 + 0.5 * g0);
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Persistent over tiles of kTetsPerCta tets.  While tile t is computed, the records and
// node coordinates of tile t+1 are in flight (cp.async into the other shared stage) and the
// node ids of tile t+2 are being loaded into registers, so the dependent tet -> coordinate
// gather and the record staging leave the critical path.
__global__ void __launch_bounds__(kElemThreads, 8)
    asm_element_kernel(int n_tets, const int4* __restrict__ tets, const double* __restrict__ coords,
                       const double* __restrict__ resp, long long stride, double* __restrict__ fe,
                       double* __restrict__ ke, unsigned long long* __restrict__ err) {
  __shared__ double s_resp[2][kTetsPerCta][42];
  __shared__ double s_x[2][kTetsPerCta][12];
  __shared__ double s_geo[kTetsPerCta][14];  // grad[4][3], volume, finite flag
  __shared__ __align__(16) double s_ke[kTetsPerCta * kKeStride];
  __shared__ int s_cbad[2][kTetsPerCta];  // per stage: some C entry of the tet is not finite
  const int le = threadIdx.x / 12, r = threadIdx.x % 12;
  if (threadIdx.x < 2 * kTetsPerCta) s_cbad[threadIdx.x / kTetsPerCta][threadIdx.x % kTetsPerCta] = 0;
  const long long n_tiles = (static_cast<long long>(n_tets) + kTetsPerCta - 1) / kTetsPerCta;
  const long long step = gridDim.x;
  // thread (le, r) fetches coordinate r % 3 of tet node r / 3
  auto node_of = [&](long long tile) -> int {
    const long long e = tile * kTetsPerCta + le;
    return (tile < n_tiles && e < n_tets) ? reinterpret_cast<const int*>(tets + e)[r / 3] : -1;
  };
  auto issue = [&](long long tile, int st, int nd) {
    if (tile >= n_tiles) return;
    const long long e0 = tile * kTetsPerCta;
    const int n_here = static_cast<int>(min(static_cast<long long>(kTetsPerCta), n_tets - e0));
    for (int i = threadIdx.x; i < n_here * 42; i += kElemThreads)
      cp_async8(&s_resp[st][i / 42][i % 42], resp + (e0 + i / 42) * stride + i % 42);
    if (nd >= 0) cp_async8(&s_x[st][le][r], coords + 3LL * nd + r % 3);
  };
  long long tile = blockIdx.x;
  int nd_next = node_of(tile + step);
  issue(tile, 0, node_of(tile));
  cp_async_commit();
  for (int st = 0; tile < n_tiles; tile += step, st ^= 1) {
    cp_async_wait_all();
    __syncthreads();  // tile's stage landed; every thread is done with the previous tile
    const int nd_after = node_of(tile + 2 * step);  // consumed next iteration
    issue(tile + step, st ^ 1, nd_next);
    cp_async_commit();
    nd_next = nd_after;
    const long long e0 = tile * kTetsPerCta;
    const int n_here = static_cast<int>(min(static_cast<long long>(kTetsPerCta), n_tets - e0));
    const long long e = e0 + le;
    const bool live = le < n_here;
    const double* sg = s_resp[st][le];  // SymTensor3 xx yy zz yz xz xy, then Mandel66
    const double* cm = sg + 6;
    if (r == 0) s_cbad[st ^ 1][le] = 0;  // next tile's flags (read after two barriers)
    if (live && !(isfinite(cm[r]) && isfinite(cm[r + 12]) && isfinite(cm[r + 24])))
      s_cbad[st][le] = 1;
    if (live && r == 0) {  // b_matrix once per element, then the error order of :118-132
      double grad[12], vol;
      const double det = tet_geom(s_x[st][le], grad, &vol);
#pragma unroll
      for (int i = 0; i < 12; ++i) s_geo[le][i] = grad[i];
      s_geo[le][12] = vol;
      const double m[6] = {sg[0], sg[1], sg[2], kSqrt2 * sg[3], kSqrt2 * sg[4], kSqrt2 * sg[5]};
      bool fin = true;
#pragma unroll
      for (int i = 0; i < 6; ++i) fin = fin && isfinite(m[i]);
      const int code = !fin ? FIBRA_E_ASM_STRESS : (!(det > 0) ? FIBRA_E_KINEMATICS : 0);
      if (code) atomicMin(err, (static_cast<unsigned long long>(e) << 8) | code);
      s_geo[le][13] = fin ? 1.0 : 0.0;  // sigma finite (C: s_cbad, after the barrier)
    }
    __syncthreads();
    // thread r owns column c = r = 3 b + bx of K_e: (C B)[:, c] stays in registers and the
    // 12 rows are produced from the register copy of grad (row indices unrolled)
    const double* grad_s = s_geo[le];
    double* kb = s_ke + le * kKeStride;
    if (live) {
      const int c = r, b = c / 3, bx = c % 3;
      const double vol = grad_s[12];
      double g[12];
  #pragma unroll
      for (int i = 0; i < 12; ++i) g[i] = grad_s[i];
      const double sig[6] = {sg[0], sg[1], sg[2], kSqrt2 * sg[3], kSqrt2 * sg[4], kSqrt2 * sg[5]};
      const double sf[9] = {sg[0], sg[5], sg[4], sg[5], sg[1], sg[3], sg[4], sg[3], sg[2]};
      const double gb[3] = {grad_s[3 * b], grad_s[3 * b + 1], grad_s[3 * b + 2]};
      double gsg[4];
  #pragma unroll
      for (int a = 0; a < 4; ++a) {
        double t = 0;  // geometric part (:160-168), i = a, j = b
  #pragma unroll
        for (int p = 0; p < 3; ++p)
  #pragma unroll
          for (int q = 0; q < 3; ++q) t += g[3 * a + p] * sf[3 * p + q] * gb[q];
        gsg[a] = t * vol;
      }
      // sigma and C finite: the structural-zero skip below is exact
    bool finite = grad_s[13] != 0.0 && !s_cbad[st][le];
      double cb[6];
      if (finite) {  // structural zeros of B skipped (exact, see b_column_sparse)
        int rc_[3];
        double vc[3];
        b_column_sparse(grad_s, c, rc_, vc);
        double s = 0;  // internal force (:137-142)
  #pragma unroll
        for (int k = 0; k < 3; ++k) s += vc[k] * sel6(sig, rc_[k]);
        fe[e * 12 + c] = vol * s;
  #pragma unroll
        for (int p = 0; p < 6; ++p) {  // C B, column c (:145-150)
          double t = 0;
  #pragma unroll
          for (int k = 0; k < 3; ++k) t += cm[6 * p + rc_[k]] * vc[k];
          cb[p] = t;
        }
  #pragma unroll
        for (int p = 0; p < 6; ++p) finite = finite && isfinite(cb[p]);
      } else {
        double bc[6];
        b_column(grad_s, c, bc);
        double s = 0;
  #pragma unroll
        for (int p = 0; p < 6; ++p) s += bc[p] * sig[p];
        fe[e * 12 + c] = vol * s;
  #pragma unroll
        for (int p = 0; p < 6; ++p) {
          double t = 0;
  #pragma unroll
          for (int q = 0; q < 6; ++q) t += cm[6 * p + q] * bc[q];
          cb[p] = t;
        }
      }
      if (finite) {
  #pragma unroll
        for (int a = 0; a < 4; ++a)
  #pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            // rows of B column 3a+ax (compile-time after unrolling): ax 0 -> 0,4,5 ...
            const double gx = g[3 * a + ax];
            const double h0 = ax == 0 ? g[3 * a + 2] : (ax == 1 ? g[3 * a + 2] : g[3 * a + 1]);
            const double h1 = ax == 0 ? g[3 * a + 1] : g[3 * a];
            const int p1 = ax == 0 ? 4 : 3, p2 = ax == 2 ? 4 : 5;
            double t = 0;  // V B^T C B (:151-157)
            t += (0.0 + gx) * cb[ax];
            t += (0.0 + kSqrt2 * (0.0 + 0.5 * h0)) * cb[p1];
            t += (0.0 + kSqrt2 * (0.0 + 0.5 * h1)) * cb[p2];
            double k = vol * t;
            if (bx == ax) k += gsg[a];
            kb[((b * 4 + a) * 3 + ax) * 3 + bx] = k;
          }
      } else {
  #pragma unroll
        for (int a = 0; a < 4; ++a)
  #pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            double br[6];
            b_column(g, 3 * a + ax, br);
            double t = 0;
  #pragma unroll
            for (int p = 0; p < 6; ++p) t += br[p] * cb[p];
            double k = vol * t;
            if (bx == ax) k += gsg[a];
            kb[((b * 4 + a) * 3 + ax) * 3 + bx] = k;
          }
      }
    }
    __syncthreads();
    // 16-byte copy-out: K_e rows are 1152 B in HBM, 1168 B (padded) in shared memory
    double2* out = reinterpret_cast<double2*>(ke + e0 * 144);
    for (int i = threadIdx.x; i < n_here * 72; i += kElemThreads)
      out[i] = *reinterpret_cast<const double2*>(&s_ke[(i / 72) * kKeStride + 2 * (i % 72)]);
  }
  cp_async_wait_all();
}

// one thread per (node pair, row axis): A row node, B column node, row dof 3 A + ax;
// contrib = e << 4 | a << 2 | b.  Three threads per pair keep more block loads in flight.
__global__ void asm_pair_kernel(long long n_pairs, const int* __restrict__ pair_a,
                                const int* __restrict__ pair_b, const int* __restrict__ pair_rowoff,
                                const long long* __restrict__ pair_ptr,
                                const unsigned* __restrict__ contrib, const int* __restrict__ fod,
                                const long long* __restrict__ col_ptr, const double* __restrict__ ke,
                                double* __restrict__ values) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long p = t / 3;
  const int ax = static_cast<int>(t % 3);
  if (p >= n_pairs) return;
  const int A = pair_a[p];
  if (fod[3 * A + ax] < 0) return;
  const int B = pair_b[p];
  const long long k0 = pair_ptr[p], k1 = pair_ptr[p + 1];
  double acc[3];
  {
    const unsigned c = contrib[k0];
    const double* row = ke + (static_cast<long long>(c >> 4) * 16 + (c & 3) * 4 + ((c >> 2) & 3)) * 9 + 3 * ax;
#pragma unroll
    for (int i = 0; i < 3; ++i) acc[i] = row[i];  // setFromTriplets: the first value as is
  }
  for (long long k = k0 + 1; k < k1; ++k) {
    const unsigned c = contrib[k];
    const double* row = ke + (static_cast<long long>(c >> 4) * 16 + (c & 3) * 4 + ((c >> 2) & 3)) * 9 + 3 * ax;
#pragma unroll
    for (int i = 0; i < 3; ++i) acc[i] = acc[i] + row[i];  // collapseDuplicates, triplet order
  }
  int before = 0;  // free row dofs of A ahead of this one in the column
  for (int i = 0; i < ax; ++i) before += fod[3 * A + i] >= 0;
  const long long off = pair_rowoff[p] + before;
#pragma unroll
  for (int bx = 0; bx < 3; ++bx) {
    const int cf = fod[3 * B + bx];
    if (cf >= 0) values[col_ptr[cf] + off] = acc[bx];
  }
}

// one thread per node with a free dof; ne = e << 2 | a, elements ascending (:170-175, :185)
__global__ void asm_residual_kernel(int n_nodes, const int* __restrict__ ne_ptr,
                                    const unsigned* __restrict__ ne, const int* __restrict__ fod,
                                    const double* __restrict__ fe, const double* __restrict__ f_ext,
                                    double* __restrict__ residual, int* __restrict__ nonfinite) {
  const int A = blockIdx.x * blockDim.x + threadIdx.x;
  if (A >= n_nodes) return;
  const int fa[3] = {fod[3 * A], fod[3 * A + 1], fod[3 * A + 2]};
  if (fa[0] < 0 && fa[1] < 0 && fa[2] < 0) return;
  double r[3] = {0.0, 0.0, 0.0};  // VectorXd::Zero
  for (int k = ne_ptr[A]; k < ne_ptr[A + 1]; ++k) {
    const unsigned c = ne[k];
    const double* f = fe + static_cast<long long>(c >> 2) * 12 + (c & 3) * 3;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) r[ax] += f[ax];
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (fa[ax] < 0) continue;
    const double v = r[ax] - (f_ext ? f_ext[fa[ax]] : 0.0);
    residual[fa[ax]] = v;
    if (!isfinite(v)) atomicExch(nonfinite, 1);
  }
}

}  // namespace

struct fibra_assembly {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  int n_tets = 0, n_nodes = 0, n_free = 0, n_sm = 148;
  long long nnz = 0, n_pairs = 0;
  std::vector<long long> col_ptr;
  std::vector<int> row_idx;
  std::string err;
  // device plan
  int4* d_tets = nullptr;
  int* d_fod = nullptr;
  long long* d_col_ptr = nullptr;
  int *d_pair_a = nullptr, *d_pair_b = nullptr, *d_pair_rowoff = nullptr;
  long long* d_pair_ptr = nullptr;
  unsigned* d_contrib = nullptr;
  int* d_ne_ptr = nullptr;
  unsigned* d_ne = nullptr;
  // per-call buffers
  double *d_fe = nullptr, *d_ke = nullptr;
  unsigned long long* d_err = nullptr;
  int* d_nonfinite = nullptr;
  double *d_coords = nullptr, *d_resp = nullptr, *d_fext = nullptr, *d_residual = nullptr,
         *d_values = nullptr;
  long long resp_cap = 0;
  cudaEvent_t ev[4] = {};
  int bad_element = -1;
};

namespace {

int as_fail(fibra_assembly* as, int code, const std::string& what) {
  if (as) as->err = what;
  return code;
}

#define AS_CUDA(as, call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return as_fail(as, FIBRA_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
int upload(fibra_assembly* as, T** dst, const T* src, size_t n) {
  AS_CUDA(as, cudaMalloc(dst, sizeof(T) * std::max<size_t>(n, 1)));
  if (n) AS_CUDA(as, cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return FIBRA_OK;
}

}  // namespace

extern "C" {

int fibra_cuda_assembly_create(int device, const int32_t* tets, int32_t n_tets, int32_t n_nodes,
                               const int32_t* free_of_dof, int32_t n_free, fibra_assembly** out) {
  if (!out || n_tets < 0 || n_nodes < 0 || n_free < 0 || (n_tets && !tets) ||
      (n_nodes && !free_of_dof))
    return FIBRA_E_ARG;
  *out = nullptr;
  if (static_cast<long long>(n_tets) >= (1LL << 28)) return FIBRA_E_ARG;  // contrib encoding
  for (long long i = 0; i < 4LL * n_tets; ++i)
    if (tets[i] < 0 || tets[i] >= n_nodes) return FIBRA_E_ARG;
  // the compressed column pattern below assumes the free slots are exactly 0..n_free-1 in
  // ascending DOF order (build_numbering, macrofem.cpp:22-38): rows then ascend in every
  // column and no two DOFs share a slot
  {
    int32_t next = 0;
    for (long long d = 0; d < 3LL * n_nodes; ++d) {
      const int32_t f = free_of_dof[d];
      if (f < 0) continue;
      if (f != next) return FIBRA_E_ARG;
      ++next;
    }
    if (next != n_free) return FIBRA_E_ARG;
  }
  auto* as = new fibra_assembly();
  as->device = device;
  as->n_tets = n_tets, as->n_nodes = n_nodes, as->n_free = n_free;
  // node -> (element, local index), elements ascending (counting sort over element order)
  std::vector<int> ne_ptr(n_nodes + 1, 0);
  for (long long i = 0; i < 4LL * n_tets; ++i) ne_ptr[tets[i] + 1]++;
  for (int v = 0; v < n_nodes; ++v) ne_ptr[v + 1] += ne_ptr[v];
  std::vector<unsigned> ne(ne_ptr[n_nodes]);
  {
    std::vector<int> fill(ne_ptr.begin(), ne_ptr.end() - 1);
    for (int e = 0; e < n_tets; ++e)
      for (int a = 0; a < 4; ++a)
        ne[fill[tets[4 * e + a]]++] = (static_cast<unsigned>(e) << 2) | a;
  }
  auto nfree = [&](int v) {
    return (free_of_dof[3 * v] >= 0) + (free_of_dof[3 * v + 1] >= 0) + (free_of_dof[3 * v + 2] >= 0);
  };
  // column node B: its row nodes A ascending, each with the shared elements ascending --
  // exactly the triplets of macrofem.cpp:170-183 grouped by (column, row) in triplet order
  std::vector<int> pa, pb, prow;
  std::vector<long long> pptr{0};
  std::vector<unsigned> contrib;
  std::vector<long long> rows_of_node(n_nodes, 0);
  std::vector<std::vector<int>> rows_list;  // per column node with free dofs: row dofs
  as->col_ptr.assign(static_cast<size_t>(n_free) + 1, 0);
  std::vector<int> col_node_rows_begin(n_nodes, -1);
  std::vector<int> row_pool;
  std::vector<std::pair<int, unsigned>> ent;  // (A, contrib) for one B
  for (int B = 0; B < n_nodes; ++B) {
    if (!nfree(B)) continue;
    ent.clear();
    for (int k = ne_ptr[B]; k < ne_ptr[B + 1]; ++k) {
      const unsigned e = ne[k] >> 2, b = ne[k] & 3;
      for (int a = 0; a < 4; ++a)
        ent.emplace_back(tets[4 * e + a], (e << 4) | (static_cast<unsigned>(a) << 2) | b);
    }
    std::stable_sort(ent.begin(), ent.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    col_node_rows_begin[B] = static_cast<int>(row_pool.size());
    int rowoff = 0;
    for (size_t i = 0; i < ent.size();) {
      size_t j = i;
      while (j < ent.size() && ent[j].first == ent[i].first) ++j;
      const int A = ent[i].first;
      if (nfree(A)) {
        pa.push_back(A), pb.push_back(B), prow.push_back(rowoff);
        for (size_t k = i; k < j; ++k) contrib.push_back(ent[k].second);
        pptr.push_back(static_cast<long long>(contrib.size()));
        for (int ax = 0; ax < 3; ++ax)
          if (free_of_dof[3 * A + ax] >= 0) row_pool.push_back(free_of_dof[3 * A + ax]);
        rowoff += nfree(A);
      }
      i = j;
    }
    rows_of_node[B] = rowoff;
  }
  // compressed column-major pattern (free numbering is ascending in dof order)
  for (int d = 0; d < 3 * n_nodes; ++d) {
    const int cf = free_of_dof[d];
    if (cf >= 0) as->col_ptr[cf + 1] = rows_of_node[d / 3];
  }
  for (int c = 0; c < n_free; ++c) as->col_ptr[c + 1] += as->col_ptr[c];
  as->nnz = as->col_ptr[n_free];
  as->row_idx.resize(as->nnz);
  for (int d = 0; d < 3 * n_nodes; ++d) {
    const int cf = free_of_dof[d];
    if (cf < 0) continue;
    const int B = d / 3;
    std::copy(row_pool.begin() + col_node_rows_begin[B],
              row_pool.begin() + col_node_rows_begin[B] + rows_of_node[B],
              as->row_idx.begin() + as->col_ptr[cf]);
  }
  as->n_pairs = static_cast<long long>(pa.size());
  int rc;
  if (cudaSetDevice(device) != cudaSuccess) { delete as; return FIBRA_E_CUDA; }
  cudaDeviceGetAttribute(&as->n_sm, cudaDevAttrMultiProcessorCount, device);
  std::vector<int4> t4(n_tets);
  for (int e = 0; e < n_tets; ++e)
    t4[e] = make_int4(tets[4 * e], tets[4 * e + 1], tets[4 * e + 2], tets[4 * e + 3]);
  if ((rc = upload(as, &as->d_tets, t4.data(), t4.size())) ||
      (rc = upload(as, &as->d_fod, free_of_dof, 3 * static_cast<size_t>(n_nodes))) ||
      (rc = upload(as, &as->d_col_ptr, as->col_ptr.data(), as->col_ptr.size())) ||
      (rc = upload(as, &as->d_pair_a, pa.data(), pa.size())) ||
      (rc = upload(as, &as->d_pair_b, pb.data(), pb.size())) ||
      (rc = upload(as, &as->d_pair_rowoff, prow.data(), prow.size())) ||
      (rc = upload(as, &as->d_pair_ptr, pptr.data(), pptr.size())) ||
      (rc = upload(as, &as->d_contrib, contrib.data(), contrib.size())) ||
      (rc = upload(as, &as->d_ne_ptr, ne_ptr.data(), ne_ptr.size())) ||
      (rc = upload(as, &as->d_ne, ne.data(), ne.size()))) {
    fibra_cuda_assembly_free(as);
    return rc;
  }
  const size_t nt = std::max(1, n_tets);
  if (cudaMalloc(&as->d_fe, sizeof(double) * 12 * nt) != cudaSuccess ||
      cudaMalloc(&as->d_ke, sizeof(double) * 144 * nt) != cudaSuccess ||
      cudaMalloc(&as->d_err, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&as->d_nonfinite, sizeof(int)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&as->stream, cudaStreamNonBlocking) != cudaSuccess) {
    fibra_cuda_assembly_free(as);
    return FIBRA_E_CUDA;
  }
  for (auto& ev : as->ev) cudaEventCreate(&ev);
  *out = as;
  return FIBRA_OK;
}

int fibra_cuda_assembly_set_stream(fibra_assembly* as, void* stream) {
  if (!as) return FIBRA_E_ARG;
  if (as->own_stream && as->stream) cudaStreamDestroy(as->stream);
  as->own_stream = stream == nullptr;
  if (stream) as->stream = static_cast<cudaStream_t>(stream);
  else AS_CUDA(as, cudaStreamCreateWithFlags(&as->stream, cudaStreamNonBlocking));
  return FIBRA_OK;
}

int fibra_cuda_assembly_pattern(const fibra_assembly* as, int64_t* nnz, int64_t* col_ptr,
                                int32_t* row_idx) {
  if (!as) return FIBRA_E_ARG;
  if (nnz) *nnz = as->nnz;
  if (col_ptr) std::copy(as->col_ptr.begin(), as->col_ptr.end(), col_ptr);
  if (row_idx) std::copy(as->row_idx.begin(), as->row_idx.end(), row_idx);
  return FIBRA_OK;
}

int fibra_cuda_assemble_device(fibra_assembly* as, const double* coords_dev,
                               const double* responses_dev, int64_t response_stride,
                               const double* f_ext_dev, double* residual_dev,
                               double* values_dev) {
  if (!as || response_stride < 42 || (as->n_tets && (!coords_dev || !responses_dev)) ||
      (as->n_free && !residual_dev) || (as->nnz && !values_dev))
    return FIBRA_E_ARG;
  AS_CUDA(as, cudaSetDevice(as->device));
  AS_CUDA(as, cudaMemsetAsync(as->d_err, 0xff, sizeof(unsigned long long), as->stream));
  AS_CUDA(as, cudaMemsetAsync(as->d_nonfinite, 0, sizeof(int), as->stream));
  cudaEventRecord(as->ev[0], as->stream);
  if (as->n_tets) {
    const long long tiles = (as->n_tets + kTetsPerCta - 1) / kTetsPerCta;
    const unsigned grid = static_cast<unsigned>(std::min<long long>(tiles, 8LL * as->n_sm));
    asm_element_kernel<<<grid, kElemThreads, 0, as->stream>>>(
        as->n_tets, as->d_tets, coords_dev, responses_dev, response_stride, as->d_fe, as->d_ke,
        as->d_err);
    AS_CUDA(as, cudaGetLastError());
  }
  cudaEventRecord(as->ev[1], as->stream);
  if (as->n_pairs) {
    asm_pair_kernel<<<static_cast<unsigned>((3 * as->n_pairs + 255) / 256), 256, 0, as->stream>>>(
        as->n_pairs, as->d_pair_a, as->d_pair_b, as->d_pair_rowoff, as->d_pair_ptr,
        as->d_contrib, as->d_fod, as->d_col_ptr, as->d_ke, values_dev);
    AS_CUDA(as, cudaGetLastError());
  }
  cudaEventRecord(as->ev[2], as->stream);
  if (as->n_nodes && as->n_free) {
    asm_residual_kernel<<<(as->n_nodes + 255) / 256, 256, 0, as->stream>>>(
        as->n_nodes, as->d_ne_ptr, as->d_ne, as->d_fod, as->d_fe, f_ext_dev, residual_dev,
        as->d_nonfinite);
    AS_CUDA(as, cudaGetLastError());
  }
  cudaEventRecord(as->ev[3], as->stream);
  return FIBRA_OK;
}

int fibra_cuda_assembly_status(fibra_assembly* as, int32_t* bad_element) {
  if (!as) return FIBRA_E_ARG;
  unsigned long long err = 0;
  int nonfinite = 0;
  AS_CUDA(as, cudaMemcpyAsync(&err, as->d_err, sizeof(err), cudaMemcpyDeviceToHost, as->stream));
  AS_CUDA(as, cudaMemcpyAsync(&nonfinite, as->d_nonfinite, sizeof(int), cudaMemcpyDeviceToHost,
                              as->stream));
  AS_CUDA(as, cudaStreamSynchronize(as->stream));
  if (bad_element) *bad_element = -1;
  if (err != ~0ULL) {
    if (bad_element) *bad_element = static_cast<int32_t>(err >> 8);
    const int code = static_cast<int>(err & 0xff);
    return as_fail(as, code, "element " + std::to_string(err >> 8) +
                                 (code == FIBRA_E_KINEMATICS ? ": inverted tetrahedron"
                                                             : ": non-finite stress response"));
  }
  if (nonfinite) return as_fail(as, FIBRA_E_ASM_RESIDUAL, "non-finite assembled residual");
  return FIBRA_OK;
}

int fibra_cuda_assemble(fibra_assembly* as, const double* coords, const double* responses,
                        int64_t response_stride, const double* f_ext_free, double* residual,
                        double* values, int32_t* bad_element) {
  if (!as || response_stride < 42 || (as->n_tets && (!coords || !responses)) ||
      (as->n_free && !residual) || (as->nnz && !values))
    return FIBRA_E_ARG;
  AS_CUDA(as, cudaSetDevice(as->device));
  if (!as->d_coords) {
    AS_CUDA(as, cudaMalloc(&as->d_coords, sizeof(double) * 3 * std::max(1, as->n_nodes)));
    AS_CUDA(as, cudaMalloc(&as->d_fext, sizeof(double) * std::max(1, as->n_free)));
    AS_CUDA(as, cudaMalloc(&as->d_residual, sizeof(double) * std::max(1, as->n_free)));
    AS_CUDA(as, cudaMalloc(&as->d_values, sizeof(double) * std::max<long long>(1, as->nnz)));
  }
  // the record array travels as one contiguous copy (a pitched 2D copy of 42-double rows
  // runs row by row); the kernel reads sigma + C at the caller's stride
  const long long rec_doubles = static_cast<long long>(response_stride) * as->n_tets;
  if (rec_doubles > as->resp_cap) {
    if (as->d_resp) cudaFree(as->d_resp);
    as->d_resp = nullptr;
    AS_CUDA(as, cudaMalloc(&as->d_resp, sizeof(double) * std::max(1LL, rec_doubles)));
    as->resp_cap = rec_doubles;
  }
  AS_CUDA(as, cudaMemcpyAsync(as->d_coords, coords, sizeof(double) * 3 * as->n_nodes,
                              cudaMemcpyHostToDevice, as->stream));
  AS_CUDA(as, cudaMemcpyAsync(as->d_resp, responses, sizeof(double) * rec_doubles,
                              cudaMemcpyHostToDevice, as->stream));
  if (f_ext_free)
    AS_CUDA(as, cudaMemcpyAsync(as->d_fext, f_ext_free, sizeof(double) * as->n_free,
                                cudaMemcpyHostToDevice, as->stream));
  int rc = fibra_cuda_assemble_device(as, as->d_coords, as->d_resp, response_stride,
                                      f_ext_free ? as->d_fext : nullptr, as->d_residual,
                                      as->d_values);
  if (rc) return rc;
  AS_CUDA(as, cudaMemcpyAsync(residual, as->d_residual, sizeof(double) * as->n_free,
                              cudaMemcpyDeviceToHost, as->stream));
  AS_CUDA(as, cudaMemcpyAsync(values, as->d_values, sizeof(double) * as->nnz,
                              cudaMemcpyDeviceToHost, as->stream));
  return fibra_cuda_assembly_status(as, bad_element);
}

int fibra_cuda_assembly_times(fibra_assembly* as, float* ms) {
  if (!as || !ms) return FIBRA_E_ARG;
  AS_CUDA(as, cudaEventSynchronize(as->ev[3]));
  for (int i = 0; i < 3; ++i) AS_CUDA(as, cudaEventElapsedTime(&ms[i], as->ev[i], as->ev[i + 1]));
  return FIBRA_OK;
}

int fibra_cuda_assembly_info(const fibra_assembly* as, int64_t* out) {
  if (!as || !out) return FIBRA_E_ARG;
  out[0] = as->n_tets, out[1] = as->n_nodes, out[2] = as->n_free, out[3] = as->nnz;
  out[4] = as->n_pairs;
  return FIBRA_OK;
}

const char* fibra_cuda_assembly_last_error(const fibra_assembly* as) {
  return as ? as->err.c_str() : "null assembly";
}

int fibra_cuda_assembly_free(fibra_assembly* as) {
  if (!as) return FIBRA_OK;
  cudaSetDevice(as->device);
  void* bufs[] = {as->d_tets, as->d_fod, as->d_col_ptr, as->d_pair_a, as->d_pair_b,
                  as->d_pair_rowoff, as->d_pair_ptr, as->d_contrib, as->d_ne_ptr, as->d_ne,
                  as->d_fe, as->d_ke, as->d_err, as->d_nonfinite, as->d_coords, as->d_resp,
                  as->d_fext, as->d_residual, as->d_values};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& ev : as->ev)
    if (ev) cudaEventDestroy(ev);
  if (as->own_stream && as->stream) cudaStreamDestroy(as->stream);
  delete as;
  return FIBRA_OK;
}

}  // extern "C"
