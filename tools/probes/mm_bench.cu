// Probe: smem matmul variants (n x n, ld = n rounded to 4), one CTA.
#include <cstdio>
#include <cuda_runtime.h>

template <int NT>
__device__ void mm_strip(const double* A, const double* B, double* C, int n, int ld) {
  const int ns = (n + 3) >> 2;
  for (int s = threadIdx.x; s < n * ns; s += NT) {
    const int i = s / ns, j0 = (s - i * ns) * 4;
    const double* a = A + i * ld;
    const double* b = B + j0;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int k = 0; k < n; ++k) {
      const double av = a[k];
      const double4 bv = *reinterpret_cast<const double4*>(b + k * ld);
      c0 += av * bv.x; c1 += av * bv.y; c2 += av * bv.z; c3 += av * bv.w;
    }
    double* c = C + i * ld + j0;
    c[0] = c0; c[1] = c1; c[2] = c2; c[3] = c3;
  }
  __syncthreads();
}
template <int NT>
__device__ void mm_one(const double* A, const double* B, double* C, int n, int ld) {
  for (int s = threadIdx.x; s < n * n; s += NT) {
    const int i = s / n, j = s - i * n;
    const double* a = A + i * ld;
    double c0 = 0;
    for (int k = 0; k < n; ++k) c0 += a[k] * B[k * ld + j];
    C[i * ld + j] = c0;
  }
  __syncthreads();
}
template <int NT>
__device__ void mm_2x2(const double* A, const double* B, double* C, int n, int ld) {
  const int nb = (n + 1) >> 1;
  for (int s = threadIdx.x; s < nb * nb; s += NT) {
    const int bi = s / nb, bj = s - bi * nb;
    const int i = 2 * bi, j = 2 * bj;
    const double* a0 = A + i * ld;
    const double* a1 = A + (i + 1) * ld;
    double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
    for (int k = 0; k < n; ++k) {
      const double2 bv = *reinterpret_cast<const double2*>(B + k * ld + j);
      const double x0 = a0[k], x1 = a1[k];
      c00 += x0 * bv.x; c01 += x0 * bv.y; c10 += x1 * bv.x; c11 += x1 * bv.y;
    }
    C[i * ld + j] = c00; C[i * ld + j + 1] = c01; C[(i + 1) * ld + j] = c10; C[(i + 1) * ld + j + 1] = c11;
  }
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_mm(double* out, long long* clk, int n) {
  extern __shared__ __align__(128) double sbuf[];
  const int ld = (n + 3) & ~3;
  double *A = sbuf, *B = sbuf + n * ld + 64, *C = B + n * ld + 64;
  for (int idx = threadIdx.x; idx < n * ld; idx += NT) { A[idx] = (idx % 7) * 0.1; B[idx] = (idx % 5) * 0.2; }
  __syncthreads();
  long long t[5];
  t[0] = clock64();
  for (int r = 0; r < 10; ++r) mm_strip<NT>(A, B, C, n, ld);
  t[1] = clock64();
  for (int r = 0; r < 10; ++r) mm_one<NT>(A, B, C, n, ld);
  t[2] = clock64();
  for (int r = 0; r < 10; ++r) mm_2x2<NT>(A, B, C, n, ld);
  t[3] = clock64();
  for (int r = 0; r < 10; ++r) __syncthreads();
  t[4] = clock64();
  if (threadIdx.x == 0) for (int q = 0; q < 4; ++q) clk[q] = (t[q + 1] - t[q]) / 10;
  if (threadIdx.x == 0) out[0] = C[5];
}
template <int NT>
void run(int n) {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  size_t sm = (3 * n * ((n + 3) & ~3) + 256) * 8;
  cudaFuncSetAttribute(k_mm<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_mm<NT><<<1, NT, sm>>>(o, c, n);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("NT=%4d n=%d %s: strip %lld  one %lld  2x2 %lld  sync %lld clk (ideal %d)\n", NT, n, cudaGetErrorString(e),
         h[0], h[1], h[2], h[3], n * n * n / 64);
}
int main() { run<1024>(42); run<512>(42); run<256>(42); run<1024>(64); run<256>(64); return 0; }
