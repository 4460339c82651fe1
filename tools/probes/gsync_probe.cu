// Probe: cost of a grid barrier and of 5-value deterministic grid reductions on
// 296 x 256-thread cooperative CTAs (mode 0: eik_dev.cuh's grid_reduce, now
// value-major; 1: grid.sync alone; 2: last-arriver reduction; 3/7: value-major
// variants; 6: barrier + one partial load).  Measured: CTA-major partials
// (round-1 baseline) 4.4 us, value-major 2.5 us, grid.sync 1.25 us.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o gsync_probe gsync_probe.cu
#include "../../paper_1805_02144_b200/csrc/eik_dev.cuh"
#include <cstdio>
using namespace eik;
// barrier + deterministic all-reduce: the last CTA to arrive sums the
// partials in CTA order and publishes the totals
template <int NV>
__device__ void grid_allreduce(Smem& sm, double (&v)[NV], double* part, unsigned* bar,
                               double* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) sm.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = 0.0;
    if (lane < NV) {
#pragma unroll
      for (int q = 0; q < NWARP; ++q) s += sm.red[q][lane];
      __stcg(part + (int64_t)blockIdx.x * NPART + lane, s);
    }
    unsigned gen = 0, last = 0;
    if (lane == 0) {
      gen = *(volatile unsigned*)(bar + 1);
      __threadfence();
      last = atomicAdd(bar, 1u) == gridDim.x - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    gen = __shfl_sync(0xffffffffu, gen, 0);
    if (last) {
      __threadfence();
      double t[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) t[k] = 0.0;
      // lanes take CTAs b = lane, lane+32, ...; then a fixed-order tree
      for (int b = lane; b < (int)gridDim.x; b += 32)
#pragma unroll
        for (int k = 0; k < NV; ++k) t[k] += __ldcg(part + (int64_t)b * NPART + k);
#pragma unroll
      for (int k = 0; k < NV; ++k) t[k] = warp_sum(t[k]);
      if (lane < NV) {
        double tk = t[0];
#pragma unroll
        for (int k = 1; k < NV; ++k) if (lane == k) tk = t[k];
        __stcg(tot + lane, tk);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicExch(bar, 0u);
        atomicAdd(bar + 1, 1u);
      }
    } else if (lane == 0) {
      while (*(volatile unsigned*)(bar + 1) == gen) { }
      __threadfence();
    }
    __syncwarp();
    if (lane < NV) sm.tot[lane] = __ldcg(tot + lane);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sm.tot[k];
  __syncthreads();
}
template <int NV>
__device__ void grid_reduce2(cg::grid_group& grid, Smem& sm, double (&v)[NV], double* part) {
  static_assert(NV <= NWARP, "one warp per value");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int par = sm.par;
  double* P = part + (int64_t)par * gridDim.x * NPART;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) sm.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NWARP; ++q) s += sm.red[q][threadIdx.x];
    __stcg(P + (int64_t)blockIdx.x * NPART + threadIdx.x, s);
  }
  if (threadIdx.x == 0) sm.par = par ^ 1;
  grid.sync();
  if (w < NV) {
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(P + (int64_t)b * NPART + w);
    s = warp_sum(s);
    if (lane == 0) sm.tot[w] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sm.tot[k];
}
template <int NV>
__device__ void grid_reduce3(cg::grid_group& grid, Smem& sm, double (&v)[NV], double* part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int par = sm.par;
  double* P = part + (int64_t)par * NV * 320;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) sm.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NWARP; ++q) s += sm.red[q][threadIdx.x];
    __stcg(P + threadIdx.x * 320 + blockIdx.x, s);
  }
  if (threadIdx.x == 0) sm.par = par ^ 1;
  grid.sync();
  if (w < NV) {
    double x[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) {
      const int b = lane + 32 * q;
      x[q] = b < G ? __ldcg(P + w * 320 + b) : 0.0;
    }
    double s = ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7])) + (x[8] + x[9]);
    s = warp_sum(s);
    if (lane == 0) sm.tot[w] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sm.tot[k];
}
__global__ void __launch_bounds__(TPB, 2) k(double* part, double* out, long long* clk, int reps, int mode, unsigned* bar, double* tot) {
  __shared__ Smem sm;
  if (threadIdx.x == 0) sm.par = 0;
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    double d[5] = {1.0 * threadIdx.x + blockIdx.x, 2.0, 3.0, 4.0, (double)r};
    if (mode == 0) grid_reduce<5>(grid, sm, d, part);
    else if (mode == 1) grid.sync();
    else if (mode == 2) grid_allreduce<5>(sm, d, part, bar, tot);
    else if (mode == 3) grid_reduce2<5>(grid, sm, d, part);
    else if (mode == 7) grid_reduce3<5>(grid, sm, d, part);
    else if (mode == 6) { grid.sync(); if (threadIdx.x < 5) sm.tot[threadIdx.x] = __ldcg(part + threadIdx.x); __syncthreads(); d[0] = sm.tot[0]; }
    acc += d[0] + d[4];
  }
  long long t1 = clock64();
  if (blockIdx.x == 5 && threadIdx.x == 0) { clk[0] = t1 - t0; out[0] = acc; }
}
int main() {
  double *part, *out, *tot; long long* c; unsigned* bar;
  cudaMalloc(&part, 2 * 8 * 320 * 8 * 2); cudaMalloc(&out, 8); cudaMalloc(&c, 8); cudaMalloc(&bar, 8); cudaMalloc(&tot, 64);
  cudaMemset(bar, 0, 8);
  for (int mode = 0; mode < 8; ++mode) {
    int reps = 1000;
    void* args[] = {&part, &out, &c, &reps, &mode, &bar, &tot};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel((void*)k, 296, TPB, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k, 296, TPB, args, 0, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double o; cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.3f us per op, check %.6e\n", mode, cudaGetErrorString(e), ms * 1e3 / reps, o);
  }
}
