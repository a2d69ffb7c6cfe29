// Microbenchmark of the resident kernel's gather step (dr_kernel.cuh node phase): per lane,
// `steps` pair-steps of {prefetched int2 CSR pair, 2 x 3 LDS.64 of signed records, 6 DFMA
// chained per component}, with W warps per CTA and 1 or 2 CTAs per SM.  Prints cycles per
// step of one warp.  nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double sign_one(int e) {
  return __hiloint2double((e & static_cast<int>(0x80000000u)) | 0x3ff00000, 0);
}

template <int W>
__global__ void gather(int steps, int reps, double* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int T = W * 32, tid = threadIdx.x;
  double* G = reinterpret_cast<double*>(sm);               // 3072 records
  int2* cent = reinterpret_cast<int2*>(sm + 3072 * 24);    // [steps+1][T]
  for (int i = tid; i < 3 * 3072; i += T) G[i] = 1e-3 * (i % 97);
  for (int i = tid; i < (steps + 1) * T; i += T) {  // conflict-free half-warp pattern
    const int l = i % T, kp = i / T;
    const int r0 = (16 * (2 * kp) + (l % 16) + 32 * (l / 16)) % 3072;
    const int r1 = (16 * (2 * kp + 1) + (l % 16) + 32 * (l / 16) + 1024) % 3072;
    cent[i] = make_int2(24 * r0 | ((l & 1) << 31), 24 * r1);
  }
  __syncthreads();
  double f0 = 0, f1 = 0, f2 = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    int2 ep = cent[tid];
    for (int kp = 0; kp < steps; ++kp) {
      const int2 en = cent[(kp + 1) * T + tid];
      const double* g0 = reinterpret_cast<const double*>(sm + (ep.x & 0x7fffffff));
      const double* g1 = reinterpret_cast<const double*>(sm + (ep.y & 0x7fffffff));
      const double a0 = g0[0], a1 = g0[1], a2 = g0[2];
      const double b0 = g1[0], b1 = g1[1], b2 = g1[2];
      const double sa = sign_one(ep.x), sb = sign_one(ep.y);
      f0 = __fma_rn(sa, a0, f0);
      f1 = __fma_rn(sa, a1, f1);
      f2 = __fma_rn(sa, a2, f2);
      f0 = __fma_rn(sb, b0, f0);
      f1 = __fma_rn(sb, b1, f1);
      f2 = __fma_rn(sb, b2, f2);
      ep = en;
    }
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * T + tid] = f0 + f1 + f2;
  if (tid == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMallocManaged(&cyc, sizeof(long long));
  const int smem = 3072 * 24 + 16 * 384 * 8;
  cudaFuncSetAttribute(gather<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  for (int steps : {1, 7}) {
    gather<1><<<1, 32, smem>>>(steps, reps, out, cyc);
    cudaDeviceSynchronize();
    gather<1><<<1, 32, smem>>>(steps, reps, out, cyc);
    cudaDeviceSynchronize();
    printf("1 warp alone, %d steps: %.1f cycles/step\n", steps, double(*cyc) / reps / steps);
    for (int ctas : {148, 296}) {
      gather<12><<<ctas, 384, smem>>>(steps, reps, out, cyc);
      cudaDeviceSynchronize();
      gather<12><<<ctas, 384, smem>>>(steps, reps, out, cyc);
      cudaDeviceSynchronize();
      printf("12 warps x %d CTAs, %d steps: %.1f cycles/step\n", ctas, steps,
             double(*cyc) / reps / steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
