// Probe: cost of the dense-phase building blocks (one CTA, matrices in
// shared memory) -- matmul, LU solve and whole expm at n = 42.
#include "../../paper_1805_02144_b200/csrc/eik_dev.cuh"
#include <cstdio>
using namespace eik;

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_dense_probe(const double* Min, double* out, long long* clk, int n) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ DenseRed rs;
  const int ld = dense_ld(n);
  double* buf = reinterpret_cast<double*>(dsm);
  double* M[6];
  for (int q = 0; q < 6; ++q) M[q] = buf + q * n * ld;
  auto load = [&]() {
    for (int idx = threadIdx.x; idx < n * ld; idx += NT) {
      const int i = idx / ld, j = idx % ld;
      M[0][idx] = j < n ? Min[i * n + j] : 0.0;
      M[1][idx] = M[0][idx];
    }
    __syncthreads();
  };
  load();
  long long t0 = clock64();
  for (int r = 0; r < 10; ++r) blk_matmul<NT>(M[0], M[1], M[2], n, ld);
  long long t1 = clock64();
  for (int r = 0; r < 10; ++r) {
    load();
    for (int idx = threadIdx.x; idx < n * ld; idx += NT) M[2][idx] = M[0][idx];
    __syncthreads();
    blk_solve<NT>(rs, M[1], M[2], n, ld);
  }
  long long t2 = clock64();
  for (int r = 0; r < 10; ++r) { load(); blk_expm<NT>(rs, M, n, ld); }
  long long t3 = clock64();
  for (int r = 0; r < 10; ++r) blk_norm1<NT>(rs, M[0], n, ld);
  long long t4 = clock64();
  if (threadIdx.x == 0) { clk[0] = (t1 - t0) / 10; clk[1] = (t2 - t1) / 10; clk[2] = (t3 - t2) / 10; clk[3] = (t4 - t3) / 10; }
  if (threadIdx.x == 0) out[0] = M[2][0];
}

template <int NT>
void run(int n) {
  double* h = new double[n * n];
  for (int i = 0; i < n * n; ++i) h[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  for (int i = 0; i < n; ++i) h[i * n + i] += 2.0;
  double *d, *o; long long* c;
  cudaMalloc(&d, n * n * 8); cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  cudaMemcpy(d, h, n * n * 8, cudaMemcpyHostToDevice);
  size_t sm = 6 * n * dense_ld(n) * 8;
  cudaFuncSetAttribute(k_dense_probe<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_dense_probe<NT><<<1, NT, sm>>>(d, o, c, n);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc[4]; cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
  printf("NT=%d n=%d (%s): matmul %lld clk, solve %lld clk (incl reload), expm %lld clk, norm1 %lld clk\n", NT, n,
         cudaGetErrorString(e), hc[0], hc[1], hc[2], hc[3]);
}
int main() {
  run<1024>(42); run<256>(42); run<1024>(64); run<512>(42);
  return 0;
}
