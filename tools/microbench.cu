// Latency / throughput microbenchmarks for the DR kernel's instruction mix on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void chain_dadd(double* out, double a, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dmul(double* out, double a, long long* cyc) {
  double x = threadIdx.x + 1.0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dfma(double* out, double a, long long* cyc) {
  double x = threadIdx.x + 1.0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, a, 1e-300);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_ddiv(double* out, double a, long long* cyc) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) x = a / x;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = (t1 - t0) * 16;
}
__global__ void chain_dsqrt(double* out, double a, long long* cyc) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) x = sqrt(x) + a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = (t1 - t0) * 16;
}
__global__ void chain_lds(double* out, long long* cyc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: W warps per block, 1 block per SM, 4 independent chains per thread
__global__ void tput_dadd(double* out, double a, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) {
    x0 = x0 + a; x1 = x1 + a; x2 = x2 + a; x3 = x3 + a;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void bar_cost(double* out, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMallocManaged(&cyc, sizeof(long long));
  auto run = [&](const char* name, auto launch, double per) {
    launch();
    cudaDeviceSynchronize();
    launch();
    cudaDeviceSynchronize();
    printf("%-34s %8.2f cycles\n", name, *cyc / per);
  };
  run("DADD dependent latency", [&] { chain_dadd<<<1, 32>>>(out, 1e-3, cyc); }, N);
  run("DMUL dependent latency", [&] { chain_dmul<<<1, 32>>>(out, 1.0000001, cyc); }, N);
  run("DFMA dependent latency", [&] { chain_dfma<<<1, 32>>>(out, 1.0000001, cyc); }, N);
  run("DDIV (IEEE) dependent latency", [&] { chain_ddiv<<<1, 32>>>(out, 2.0, cyc); }, N);
  run("DSQRT+DADD dependent latency", [&] { chain_dsqrt<<<1, 32>>>(out, 0.5, cyc); }, N);
  run("LDS.32 dependent latency", [&] { chain_lds<<<1, 32>>>(out, cyc); }, N);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "DADD warp-instr / cycle / SM, %2d warps", w);
    tput_dadd<<<1, 32 * w>>>(out, 1e-3, cyc);
    cudaDeviceSynchronize();
    tput_dadd<<<1, 32 * w>>>(out, 1e-3, cyc);
    cudaDeviceSynchronize();
    printf("%-34s %8.3f\n", nm, 4.0 * N * w / *cyc);
  }
  for (int w : {4, 12, 16, 24}) {
    bar_cost<<<1, 32 * w>>>(out, cyc);
    cudaDeviceSynchronize();
    bar_cost<<<1, 32 * w>>>(out, cyc);
    cudaDeviceSynchronize();
    printf("__syncthreads, %2d warps           %8.2f cycles\n", w, *cyc / 1024.0);
  }
  return 0;
}
