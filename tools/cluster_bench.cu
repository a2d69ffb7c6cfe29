// Microbenchmark: cost of one cluster-wide barrier on B200, as the cluster DR kernel uses it
// (dr_cluster.cuh cl_sync), for C = 2..16 CTAs of 384 threads, with and without a DSMEM
// store per thread before it, release/acquire vs relaxed arrive.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bench cluster_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0 release/acquire, 1 relaxed arrive, 2 release/acquire + DSMEM store
__global__ void cl_bar(int iters, long long* cyc) {
  __shared__ double buf[384];
  unsigned rank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const unsigned me = static_cast<unsigned>(__cvta_generic_to_shared(buf + threadIdx.x));
  unsigned peer;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(me), "r"((rank + 1) % csize));
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 2) asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(peer), "d"(1.0 * i));
    if (MODE == 1)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;");
    else
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(int C, long long* cyc) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 16);
  cfg.blockDim = dim3(384);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (C > 8) cudaFuncSetAttribute(cl_bar<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 20000;
  for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, cl_bar<MODE>, iters, cyc);
  cudaDeviceSynchronize();
  printf("C=%2d mode %d: %.1f cycles per barrier (%s)\n", C, MODE, double(*cyc) / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc;
  cudaMallocManaged(&cyc, sizeof(long long));
  for (int C : {2, 4, 8, 16}) {
    run<0>(C, cyc);
    run<1>(C, cyc);
    run<2>(C, cyc);
  }
  return 0;
}
