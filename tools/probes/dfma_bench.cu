// Probe: DFMA latency/throughput and smem-operand matmul variants on one SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* clk, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  out[threadIdx.x] = a;
}
template <int CH>
__global__ void k_tput(double* out, long long* clk, int iters) {
  double a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 1.0000001, c = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  double s = 0;
  for (int k = 0; k < CH; ++k) s += a[k];
  out[threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 4096); cudaMalloc(&c, 64);
  long long h;
  k_lat<<<1, 32>>>(o, c, 4096); cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", h / 4096.0);
  for (int nt : {128, 256, 512, 1024}) {
    k_tput<8><<<1, nt>>>(o, c, 1024); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %d x 8 chains: %.2f DFMA/clk/SM\n", nt, (double)nt * 8 * 1024 / h);
  }
  return 0;
}
