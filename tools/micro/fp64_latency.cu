// Dependent-issue latency and per-SM throughput of fp64 add / mul on the GPU at hand (design input for the GICP
// step kernel's ordered sums): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, double x, int n) {
  double a = x, b = x * 0.5;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a += b;  // 16 dependent DADD
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <int ILP>
__global__ void tput(double* out, long long* cyc, double x, int n) {
  double a[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) a[q] = x + q;
  const double b = x * 0.5;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < ILP; ++q) a[q] += b;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int q = 0; q < ILP; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  long long *cyc, h;
  cudaMalloc(&out, 8 * 1024 * 1024), cudaMalloc(&cyc, 8);
  const int n = 4096;
  chain<<<1, 32>>>(out, cyc, 1.0, n), cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD latency: %.2f cycles\n", (double)h / (16.0 * n));
  for (int warps = 1; warps <= 16; warps *= 2) {
    tput<1><<<1, 32 * warps>>>(out, cyc, 1.0, n), cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d, ILP 1: %.2f DADD warp-instr / cycle / SM\n", warps, warps * 4.0 * n / (double)h);
    tput<4><<<1, 32 * warps>>>(out, cyc, 1.0, n), cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d, ILP 4: %.2f DADD warp-instr / cycle / SM\n", warps, warps * 16.0 * n / (double)h);
    tput<8><<<1, 32 * warps>>>(out, cyc, 1.0, n), cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d, ILP 8: %.2f DADD warp-instr / cycle / SM\n", warps, warps * 32.0 * n / (double)h);
  }
  return 0;
}
