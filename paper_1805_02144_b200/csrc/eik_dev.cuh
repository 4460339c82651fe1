// eik_dev.cuh -- device side of libeik (sm_100a, fp64).
//
// Execution model: every engine call (and every integrator step) runs as ONE
// cooperative persistent kernel.  The grid is sized to the co-resident
// capacity (multiple of the 148 SMs) or to the problem when that is smaller.
// Phases are separated by grid.sync(); global reductions are deterministic
// (per-CTA partials reduced in a fixed order by every CTA redundantly), so
// every CTA holds bit-identical scalars and evaluates the phipm controller
// itself -- no host round trip per substep, no broadcast needed.
//
// Vectors are "cell-interleaved": one double4 (a_x, a_y, a_z, b) per cell for
// the shallow-water operator (so one 32-byte sector per neighbour gather),
// or a zero-padded plain vector viewed as double4 units for a generic CSR
// operator.  Host <-> device conversion happens only at the C-ABI boundary.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eik.h"
#include "eik_control.h"

namespace cg = cooperative_groups;

namespace eik {

constexpr int TPB = 512;        // one CTA of 16 warps per SM (<=128 regs)
constexpr int NWARP = TPB / 32;
constexpr int NPART = 8;   // doubles per CTA partial record
constexpr int MAXV = 8;    // v_0..v_7
constexpr int MAXNS = 8;   // output points
constexpr int MAXDIM = kDenseCap;
constexpr int KMAX = 8;    // stencil slots per cell (self + up to 7)
constexpr int NOPS = 10;
// Gram-identity norm of the orthogonalised vector is used while it keeps
// h^2 > kGramSafe ||z||^2 (relative error of h below ~1e-14); else an
// explicit orthogonalisation pass recomputes it.
constexpr double kGramSafe = 1e-2;   // Gx Gy Gz Dx Dy Dz Vx Vy Vz L
enum { OP_GX = 0, OP_GY, OP_GZ, OP_DX, OP_DY, OP_DZ, OP_VX, OP_VY, OP_VZ, OP_L };

// ------------------------------------------------------------ double4 math
__device__ __forceinline__ double4 d4(double a) { return make_double4(a, a, a, a); }
__device__ __forceinline__ double4 operator+(double4 a, double4 b) {
  return make_double4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ double4 operator-(double4 a, double4 b) {
  return make_double4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
__device__ __forceinline__ double4 operator*(double s, double4 a) {
  return make_double4(s * a.x, s * a.y, s * a.z, s * a.w);
}
__device__ __forceinline__ double dot4(double4 a, double4 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}
__device__ __forceinline__ double nz4(double4 a) {
  return (double)((a.x != 0.0) + (a.y != 0.0) + (a.z != 0.0) + (a.w != 0.0));
}
__device__ __forceinline__ double nf4(double4 a) {  // count of non-finite
  return (double)(!isfinite(a.x) + !isfinite(a.y) + !isfinite(a.z) + !isfinite(a.w));
}
__device__ __forceinline__ double4 div4(double4 a, double h) {
  return make_double4(a.x / h, a.y / h, a.z / h, a.w / h);
}
// exact "p ? p[u] : 0"
__device__ __forceinline__ double4 ld4(const double4* p, int64_t u) {
  return p ? p[u] : d4(0.0);
}

// ---------------------------------------------------------------- shared
struct Smem {
  double red[NWARP][NPART];
  double tot[NPART];
  double phi[MAXDIM + 4];
  int ival[4];
  int par;  // partial-buffer parity (double buffering, see grid_reduce)
};

__device__ __forceinline__ void brange(int64_t NU, int64_t& lo, int64_t& hi) {
  int64_t G = gridDim.x, c = (NU + G - 1) / G;
  lo = (int64_t)blockIdx.x * c;
  if (lo > NU) lo = NU;
  hi = lo + c < NU ? lo + c : NU;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA partial -> part[blockIdx.x][0..NV)
template <int NV>
__device__ void part_store(Smem& sm, double (&v)[NV], double* part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = warp_sum(v[k]);
    if (lane == 0) sm.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NWARP; ++q) s += sm.red[q][threadIdx.x];
    part[(int64_t)blockIdx.x * NPART + threadIdx.x] = s;
  }
  __syncthreads();
}

// after grid.sync(): identical totals in every CTA
template <int NV>
__device__ void part_total(Smem& sm, const double* part, double (&out)[NV]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += TPB) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __ldcg(part + (int64_t)b * NPART + k);
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = warp_sum(v[k]);
    if (lane == 0) sm.red[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NWARP; ++q) s += sm.red[q][threadIdx.x];
    sm.tot[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = sm.tot[k];
  __syncthreads();
}

// Partials are double-buffered: a fast CTA may start the next reduction's
// part_store while a slow CTA still reads this one's partials; the two
// buffers alternate, and at least one grid.sync separates reuse.
template <int NV>
__device__ void grid_reduce(cg::grid_group& grid, Smem& sm, double (&v)[NV],
                            double* part) {
  const int par = sm.par;
  double* P = part + (int64_t)par * gridDim.x * NPART;
  part_store<NV>(sm, v, P);
  if (threadIdx.x == 0) sm.par = par ^ 1;
  grid.sync();
  part_total<NV>(sm, P, v);
}

// =================================================================== operators

// Shallow-water Jacobian / tendency on an unstructured stencil (ELL in the
// CSR rows' sorted column order; pads repeat the cell with zero coefficients).
struct SweOp {
  int64_t N;
  int K;
  const int* nbr;        // [K][N]
  const double* coef;    // [K][NOPS][N]
  const double4* nf;     // (n_x, n_y, n_z, f)
  const double* hs;      // surface height
  double g, nu;
  double4* lin;          // linearisation state U = (u_x, u_y, u_z, h)
  double4* ne;           // (n_x, n_y, n_z, eta) at the linearisation state
  double4* lapA;         // scratch: L x
  double4* lapB;         // scratch: second L x
  double scale;          // A x = scale * (J x)   (integrators.py:117)
  // n_A counting data
  const double* df1;     // [K][N] Df(i, slot) (0 where Df has no entry)
  const int* dfx;        // [N] nonzero Df entries outside the slot set
  const int* cnt;        // [N] valid slots
  // tiled single-pass Krylov iteration (cells tiled along the Hilbert order;
  // each tile's 2-ring halo is staged in shared memory)
  int ntiles;
  const int* t_cell0;    // first own cell
  const int* t_nT;       // own cells (<= TPB)
  const int* t_nE1;      // own + 1-ring halo
  const int* t_nE2;      // own + 1-ring + 2-ring halo
  const int* t_e2off;    // offset into e2map
  const int* t_e1off;    // offset into lnbr (rows)
  const int* e2map;      // local -> global cell id, order [own, H1, H2]
  const short* lnbr;     // [rows][8] local neighbour slots of E1 cells
  const double* Lc;      // [N][8] Laplacian row in slot order (cell-major)
  int e1max, e2max;

  static constexpr bool kTiled = true;
  __device__ __forceinline__ int64_t NU() const { return N; }
  __device__ __forceinline__ double c(int s, int op, int64_t i) const {
    return __ldg(coef + ((int64_t)s * NOPS + op) * N + i);
  }
  __device__ __forceinline__ int64_t nb(int s, int64_t i) const {
    return __ldg(nbr + (int64_t)s * N + i);
  }
};

// L x for one cell
template <class Src>
__device__ __forceinline__ double4 swe_lap_cell(const SweOp& S, const Src& x,
                                                int64_t i) {
  double4 acc = d4(0.0);
  for (int s = 0; s < S.K; ++s) {
    const int64_t j = S.nb(s, i);
    const double l = S.c(s, OP_L, i);
    const double4 xj = x(j);
    acc.x += l * xj.x;
    acc.y += l * xj.y;
    acc.z += l * xj.z;
    acc.w += l * xj.w;
  }
  return acc;
}

// (J a)(i) at the linearisation state:
//   (J a)_k = -P_k zeta_a - eta (n x a)_k - G_k e_a - nu L(L a_k)
//   (J a)_h = -sum_k D_k (h a_k + u_k b) - nu L(L b)
// zeta_a = V.a, e_a = u.a + g b.  La = L a (precomputed, gathered).
template <class Src>
__device__ __forceinline__ double4 swe_jv_cell(const SweOp& S, const Src& a,
                                               const double4* La, int64_t i) {
  double zeta = 0.0, gx = 0.0, gy = 0.0, gz = 0.0, dv = 0.0;
  double4 ll = d4(0.0);
  for (int s = 0; s < S.K; ++s) {
    const int64_t j = S.nb(s, i);
    const double4 aj = a(j);
    const double4 U = S.lin[j];
    const double4 la = La[j];
    zeta += S.c(s, OP_VX, i) * aj.x + S.c(s, OP_VY, i) * aj.y + S.c(s, OP_VZ, i) * aj.z;
    const double e = U.x * aj.x + U.y * aj.y + U.z * aj.z + S.g * aj.w;
    gx += S.c(s, OP_GX, i) * e;
    gy += S.c(s, OP_GY, i) * e;
    gz += S.c(s, OP_GZ, i) * e;
    dv += S.c(s, OP_DX, i) * (U.w * aj.x + U.x * aj.w) +
          S.c(s, OP_DY, i) * (U.w * aj.y + U.y * aj.w) +
          S.c(s, OP_DZ, i) * (U.w * aj.z + U.z * aj.w);
    const double l = S.c(s, OP_L, i);
    ll.x += l * la.x;
    ll.y += l * la.y;
    ll.z += l * la.z;
    ll.w += l * la.w;
  }
  const double4 ai = a(i);
  const double4 U = S.lin[i];
  const double4 q = S.ne[i];
  const double px = q.y * U.z - q.z * U.y;
  const double py = q.z * U.x - q.x * U.z;
  const double pz = q.x * U.y - q.y * U.x;
  const double cx = q.y * ai.z - q.z * ai.y;
  const double cy = q.z * ai.x - q.x * ai.z;
  const double cz = q.x * ai.y - q.y * ai.x;
  double4 r;
  r.x = -(px * zeta) - q.w * cx - gx - S.nu * ll.x;
  r.y = -(py * zeta) - q.w * cy - gy - S.nu * ll.y;
  r.z = -(pz * zeta) - q.w * cz - gz - S.nu * ll.z;
  r.w = -dv - S.nu * ll.w;
  return r;
}

// F(w)(i) (swe.py:149-168) with Lw = L w gathered; eta written to *eta_out
template <class Src>
__device__ __forceinline__ double4 swe_rhs_cell(const SweOp& S, const Src& w,
                                                const double4* Lw, int64_t i,
                                                double* eta_out) {
  double zeta = 0.0, gx = 0.0, gy = 0.0, gz = 0.0, dv = 0.0;
  double4 ll = d4(0.0);
  for (int s = 0; s < S.K; ++s) {
    const int64_t j = S.nb(s, i);
    const double4 wj = w(j);
    const double hsj = __ldg(S.hs + j);
    zeta += S.c(s, OP_VX, i) * wj.x + S.c(s, OP_VY, i) * wj.y + S.c(s, OP_VZ, i) * wj.z;
    const double E = 0.5 * (wj.x * wj.x + wj.y * wj.y + wj.z * wj.z) + S.g * (wj.w + hsj);
    gx += S.c(s, OP_GX, i) * E;
    gy += S.c(s, OP_GY, i) * E;
    gz += S.c(s, OP_GZ, i) * E;
    dv += S.c(s, OP_DX, i) * (wj.x * wj.w) + S.c(s, OP_DY, i) * (wj.y * wj.w) +
          S.c(s, OP_DZ, i) * (wj.z * wj.w);
    const double l = S.c(s, OP_L, i);
    const double4 lw = Lw[j];
    ll.x += l * lw.x;
    ll.y += l * lw.y;
    ll.z += l * lw.z;
    ll.w += l * lw.w;
  }
  const double4 wi = w(i);
  const double4 q = S.nf[i];
  const double eta = zeta + q.w;
  *eta_out = eta;
  const double px = q.y * wi.z - q.z * wi.y;
  const double py = q.z * wi.x - q.x * wi.z;
  const double pz = q.x * wi.y - q.y * wi.x;
  double4 r;
  r.x = -eta * px - gx - S.nu * ll.x;
  r.y = -eta * py - gy - S.nu * ll.y;
  r.z = -eta * pz - gz - S.nu * ll.z;
  r.w = -dv - S.nu * ll.w;
  return r;
}


// ------------------------------------------------------------ tiled pass
// Dynamic shared memory of one CTA: the tile's vector on E2, its Laplacian
// and the linearisation state on E1, the E2 local->global map.
struct TileSmem {
  double4* x;
  double4* La;
  double4* U;
  int* gid;
};

__device__ __forceinline__ TileSmem tile_smem(const SweOp& S) {
  extern __shared__ __align__(16) unsigned char dsm[];
  TileSmem t;
  t.x = reinterpret_cast<double4*>(dsm);
  t.La = t.x + S.e2max;
  t.U = t.La + S.e1max;
  t.gid = reinterpret_cast<int*>(t.U + S.e1max);
  return t;
}

__host__ __device__ constexpr size_t tile_smem_bytes(int e1max, int e2max) {
  return (size_t)e2max * 32 + (size_t)e1max * 64 + (size_t)e2max * 4 + 16;
}

struct Row8 {
  short s[8];
};
__device__ __forceinline__ Row8 load_row8(const short* p) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(p));
  Row8 r;
  memcpy(&r, &v, 16);
  return r;
}

// J x for own cell `c` of the tile (x, La, U staged in smem)
__device__ __forceinline__ double4 swe_jv_tile(const SweOp& S, const TileSmem& ts,
                                               const Row8& row, int c, int64_t i) {
  double zeta = 0.0, gx = 0.0, gy = 0.0, gz = 0.0, dv = 0.0;
  double4 ll = d4(0.0);
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s < S.K) {
      const int l = row.s[s];
      const double4 aj = ts.x[l];
      const double4 U = ts.U[l];
      const double4 la = ts.La[l];
      const double* cp = S.coef + (int64_t)s * NOPS * S.N + i;
      const double vx = __ldcs(cp + OP_VX * S.N), vy = __ldcs(cp + OP_VY * S.N),
                   vz = __ldcs(cp + OP_VZ * S.N);
      const double gcx = __ldcs(cp + OP_GX * S.N), gcy = __ldcs(cp + OP_GY * S.N),
                   gcz = __ldcs(cp + OP_GZ * S.N);
      const double dx = __ldcs(cp + OP_DX * S.N), dy = __ldcs(cp + OP_DY * S.N),
                   dz = __ldcs(cp + OP_DZ * S.N);
      const double l0 = __ldcs(cp + OP_L * S.N);
      zeta += vx * aj.x + vy * aj.y + vz * aj.z;
      const double e = U.x * aj.x + U.y * aj.y + U.z * aj.z + S.g * aj.w;
      gx += gcx * e;
      gy += gcy * e;
      gz += gcz * e;
      dv += dx * (U.w * aj.x + U.x * aj.w) + dy * (U.w * aj.y + U.y * aj.w) +
            dz * (U.w * aj.z + U.z * aj.w);
      ll.x += l0 * la.x;
      ll.y += l0 * la.y;
      ll.z += l0 * la.z;
      ll.w += l0 * la.w;
    }
  }
  const double4 ai = ts.x[c];
  const double4 U = ts.U[c];
  const double4 q = S.ne[i];
  const double px = q.y * U.z - q.z * U.y;
  const double py = q.z * U.x - q.x * U.z;
  const double pz = q.x * U.y - q.y * U.x;
  const double cx = q.y * ai.z - q.z * ai.y;
  const double cy = q.z * ai.x - q.x * ai.z;
  const double cz = q.x * ai.y - q.y * ai.x;
  double4 r;
  r.x = -(px * zeta) - q.w * cx - gx - S.nu * ll.x;
  r.y = -(py * zeta) - q.w * cy - gy - S.nu * ll.y;
  r.z = -(pz * zeta) - q.w * cz - gz - S.nu * ll.z;
  r.w = -dv - S.nu * ll.w;
  return r;
}

// One pass over every tile: x = form(g, own) on E2 -> smem, L x on E1,
// z = scale * J x on the own cells -> epi(i, c, z, x_i).  A whole Krylov
// iteration (orthogonalise + normalise v_j, L v_j, J v_j, projections) is
// one such pass: one HBM sweep and one grid barrier per iteration.
template <class Form, class Epi>
__device__ void swe_tiled(const SweOp& S, const Form& form, const Epi& epi) {
  const TileSmem ts = tile_smem(S);
  for (int t = blockIdx.x; t < S.ntiles; t += gridDim.x) {
    const int64_t c0 = __ldg(S.t_cell0 + t);
    const int nT = __ldg(S.t_nT + t), nE1 = __ldg(S.t_nE1 + t), nE2 = __ldg(S.t_nE2 + t);
    const int* map = S.e2map + __ldg(S.t_e2off + t);
    const short* rows = S.lnbr + (int64_t)__ldg(S.t_e1off + t) * 8;
    for (int c = threadIdx.x; c < nE2; c += TPB) {
      const int g = __ldg(map + c);
      ts.gid[c] = g;
      ts.x[c] = form(g, c < nT);
      if (c < nE1) ts.U[c] = S.lin[g];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nE1; c += TPB) {
      const Row8 row = load_row8(rows + (int64_t)c * 8);
      const double* lc = S.Lc + (int64_t)ts.gid[c] * 8;
      double4 acc = d4(0.0);
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (s < S.K) {
          const double l = __ldg(lc + s);
          const double4 xv = ts.x[row.s[s]];
          acc.x += l * xv.x;
          acc.y += l * xv.y;
          acc.z += l * xv.z;
          acc.w += l * xv.w;
        }
      }
      ts.La[c] = acc;
    }
    __syncthreads();
    if (threadIdx.x < nT) {
      const int c = threadIdx.x;
      const int64_t i = c0 + c;
      const Row8 row = load_row8(rows + (int64_t)c * 8);
      const double4 z = S.scale * swe_jv_tile(S, ts, row, c, i);
      epi(i, z, ts.x[c]);
    }
    __syncthreads();
  }
}

struct SrcPtr {
  const double4* p;
  __device__ __forceinline__ double4 operator()(int64_t j) const { return p[j]; }
};
struct SrcDiff {  // a[j] - b[j]
  const double4* a;
  const double4* b;
  __device__ __forceinline__ double4 operator()(int64_t j) const { return a[j] - b[j]; }
};

// Generic CSR operator on a zero-padded plain vector (units of 4 rows).
struct CsrOp {
  static constexpr bool kTiled = false;
  int64_t n, NUu;
  const int* rp;
  const int* ci;
  const double* val;
  double scale;
  __device__ __forceinline__ int64_t NU() const { return NUu; }
};

// ------------------------------------------------- operator "pre" + "main"
// pre: everything a matvec needs before its main phase that reads other
// CTAs' output (SWE: L x into lapA, scaled by inv).  main: (A x)(unit).

__device__ __forceinline__ void op_pre(const SweOp& S, const double4* x,
                                       double inv, int64_t lo, int64_t hi) {
  SrcPtr src{x};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB)
    S.lapA[i] = inv * swe_lap_cell(S, src, i);
}
__device__ __forceinline__ void op_pre(const CsrOp&, const double4*, double,
                                       int64_t, int64_t) {}

__device__ __forceinline__ double4 op_main(const SweOp& S, const double4* x,
                                           int64_t i) {
  return S.scale * swe_jv_cell(S, SrcPtr{x}, S.lapA, i);
}
__device__ __forceinline__ double4 op_main(const CsrOp& C, const double4* x4,
                                           int64_t u) {
  const double* x = reinterpret_cast<const double*>(x4);
  double r[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int64_t row = 4 * u + c;
    double s = 0.0;
    if (row < C.n) {
      const int b = __ldg(C.rp + row), e = __ldg(C.rp + row + 1);
      for (int k = b; k < e; ++k) s += __ldg(C.val + k) * x[__ldg(C.ci + k)];
    }
    r[c] = C.scale * s;
  }
  return make_double4(r[0], r[1], r[2], r[3]);
}

// =================================================================== dense exp
// Block-level degree-13 Pade with scaling and squaring (kernels.py:119-145),
// run by one CTA on an L2-resident scratch; LU with partial pivoting
// (LAPACK dgesv semantics: first max |pivot|, reciprocal scaling).

__device__ void blk_matmul(const double* A, const double* B, double* C, int n) {
  for (int idx = threadIdx.x; idx < n * n; idx += TPB) {
    const int i = idx / n, j = idx - i * n;
    const double* a = A + (int64_t)i * n;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += a[k] * B[(int64_t)k * n + j];
    C[idx] = s;
  }
  __syncthreads();
}

// max_j sum_i |M[i][j]|, rows summed in ascending order (numpy axis-0 reduce)
__device__ double blk_norm1(Smem& sm, const double* M, int n) {
  double best = 0.0;
  for (int j = threadIdx.x; j < n; j += TPB) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += fabs(M[(int64_t)i * n + j]);
    best = fmax(best, s);
  }
  // block max
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm.red[w][0] = best;
  __syncthreads();
  double r = 0.0;
  for (int q = 0; q < NWARP; ++q) r = fmax(r, sm.red[q][0]);
  __syncthreads();
  return r;
}

// Solve P X = Q in place (Q <- X), P overwritten by its LU factors.
__device__ void blk_solve(Smem& sm, double* P, double* Q, int n) {
  for (int k = 0; k < n; ++k) {
    // pivot: first index of max |P[i][k]|, i >= k (warp 0)
    if (threadIdx.x < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + threadIdx.x; i < n; i += 32) {
        const double v = fabs(P[(int64_t)i * n + k]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (threadIdx.x == 0) sm.ival[0] = bi;
    }
    __syncthreads();
    const int piv = sm.ival[0];
    if (piv != k) {
      for (int j = threadIdx.x; j < n; j += TPB) {
        double t = P[(int64_t)k * n + j];
        P[(int64_t)k * n + j] = P[(int64_t)piv * n + j];
        P[(int64_t)piv * n + j] = t;
        t = Q[(int64_t)k * n + j];
        Q[(int64_t)k * n + j] = Q[(int64_t)piv * n + j];
        Q[(int64_t)piv * n + j] = t;
      }
      __syncthreads();
    }
    const double pkk = P[(int64_t)k * n + k];
    const double rinv = 1.0 / pkk;
    for (int i = k + 1 + threadIdx.x; i < n; i += TPB) P[(int64_t)i * n + k] *= rinv;
    __syncthreads();
    const int rows = n - k - 1;
    const int width = (n - k - 1) + n;  // trailing P columns + all Q columns
    for (int idx = threadIdx.x; idx < rows * width; idx += TPB) {
      const int i = k + 1 + idx / width;
      const int c = idx - (idx / width) * width;
      const double l = P[(int64_t)i * n + k];
      if (c < n - k - 1) {
        const int j = k + 1 + c;
        P[(int64_t)i * n + j] -= l * P[(int64_t)k * n + j];
      } else {
        const int j = c - (n - k - 1);
        Q[(int64_t)i * n + j] -= l * Q[(int64_t)k * n + j];
      }
    }
    __syncthreads();
  }
  // back substitution (dtrsm upper, non-unit)
  for (int k = n - 1; k >= 0; --k) {
    const double pkk = P[(int64_t)k * n + k];
    for (int j = threadIdx.x; j < n; j += TPB) Q[(int64_t)k * n + j] /= pkk;
    __syncthreads();
    for (int idx = threadIdx.x; idx < k * n; idx += TPB) {
      const int i = idx / n, j = idx - i * n;
      Q[(int64_t)i * n + j] -= Q[(int64_t)k * n + j] * P[(int64_t)i * n + k];
    }
    __syncthreads();
  }
}

// E = expm(M0) for the n x n matrix in M0; returns the index of the scratch
// matrix holding E.  scratch: 6 matrices of MAXDIM^2.
__device__ int blk_expm(Smem& sm, double* scr, int n) {
  const int64_t S2 = (int64_t)MAXDIM * MAXDIM;
  double* M[6];
  for (int q = 0; q < 6; ++q) M[q] = scr + q * S2;
  const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0, 129060195264000.0, 10559470521600.0,
                        670442572800.0, 33522128640.0, 1323241920.0, 40840800.0,
                        960960.0, 16380.0, 182.0, 1.0};
  const int nn = n * n;
  const double nrm = blk_norm1(sm, M[0], n);
  int s = 0;
  if (nrm > kPadeTheta) {
    const double c = ceil(log2(nrm / kPadeTheta));
    s = c > 0.0 ? (int)c : 0;
  }
  const double sc = ldexp(1.0, s);
  if (s > 0) {
    for (int idx = threadIdx.x; idx < nn; idx += TPB) M[0][idx] = M[0][idx] / sc;
    __syncthreads();
  }
  double *X = M[0], *X2 = M[1], *X4 = M[2], *X6 = M[3];
  blk_matmul(X, X, X2, n);
  blk_matmul(X2, X2, X4, n);
  blk_matmul(X2, X4, X6, n);
  double* T = M[4];
  for (int idx = threadIdx.x; idx < nn; idx += TPB)
    T[idx] = b[13] * X6[idx] + b[11] * X4[idx] + b[9] * X2[idx];
  __syncthreads();
  double* T2 = M[5];
  blk_matmul(X6, T, T2, n);
  for (int idx = threadIdx.x; idx < nn; idx += TPB) {
    const int i = idx / n, j = idx - i * n;
    T2[idx] = T2[idx] + b[7] * X6[idx] + b[5] * X4[idx] + b[3] * X2[idx] +
              (i == j ? b[1] : 0.0);
  }
  __syncthreads();
  double* U = M[4];  // T is dead
  blk_matmul(X, T2, U, n);
  double* T3 = M[5];  // T2 is dead
  for (int idx = threadIdx.x; idx < nn; idx += TPB)
    T3[idx] = b[12] * X6[idx] + b[10] * X4[idx] + b[8] * X2[idx];
  __syncthreads();
  double* V = M[0];  // X is dead
  blk_matmul(X6, T3, V, n);
  for (int idx = threadIdx.x; idx < nn; idx += TPB) {
    const int i = idx / n, j = idx - i * n;
    const double v = V[idx] + b[6] * X6[idx] + b[4] * X4[idx] + b[2] * X2[idx] +
                     (i == j ? b[0] : 0.0);
    const double u = U[idx];
    M[1][idx] = v - u;  // P (X2 dead after this loop: read before write per idx)
    M[2][idx] = v + u;  // Q (X4 likewise)
  }
  __syncthreads();
  blk_solve(sm, M[1], M[2], n);
  int cur = 2, oth = 3;
  for (int q = 0; q < s; ++q) {
    blk_matmul(M[cur], M[cur], M[oth], n);
    const int t = cur; cur = oth; oth = t;
  }
  return cur;
}

// =================================================================== engine

struct EngineTask {
  const double4* v[MAXV];   // v_0..v_p (nullptr = zero vector)
  int p, ns;
  double rho[MAXNS];
  double tol, delta, tau_init;
  int64_t m_init, iom, m_max, max_attempts;
  int zero_skip;
  double4* W[MAXNS];
  int slot;                 // warm-start slot (-1: none)
  int info_idx;             // index into the info array
};

struct EngineWork {
  double4* basis;           // m_alloc * NU
  double4* zbuf;            // raw next Krylov vector
  double4* zbuf2;           // second z buffer (tiled path ping-pong)
  double4* w[MAXV];         // w_1..w_p
  double4* ybuf[2];
  double4* zero;            // an all-zero vector (y when v_0 == 0)
  double* part;             // [2][G][NPART]
  double* H;                // m_alloc x m_alloc
  double* scr;              // 6 * MAXDIM^2
  double* phi;              // MAXDIM + 4
  double* seeds;            // [EIK_NUM_SLOTS][2]
  EikPhipmInfo* info;       // per call
  EikTraceRec* trace;
  int64_t trace_cap;
  int64_t* trace_len;
  unsigned long long* kiters;
  int64_t NU, n, nnz, m_alloc;
};

// phipm_simul_iom2 (phipm.py:291-370); returns an eik_status, uniformly in
// every CTA.
template <class Op>
__device__ int engine_call(cg::grid_group& grid, Smem& sm, const Op& op,
                           const EngineTask& T, const EngineWork& Wk) {
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int64_t NU = Wk.NU, n = Wk.n;
  const int p = T.p;
  int64_t lo, hi;
  brange(NU, lo, hi);

  // ---- exact nonzero flags of v_l (the reference's vl.any())
  bool vnz[MAXV];
  {
    double c[NPART];
#pragma unroll
    for (int l = 0; l < NPART; ++l) c[l] = 0.0;
    for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
#pragma unroll
      for (int l = 0; l < MAXV; ++l)
        if (l <= p && T.v[l]) c[l] += nz4(T.v[l][u]);
    }
    grid_reduce<NPART>(grid, sm, c, Wk.part);
    bool any = false;
#pragma unroll
    for (int l = 0; l < MAXV; ++l) {
      vnz[l] = (l <= p) && T.v[l] && c[l] > 0.0;
      any |= vnz[l];
    }
    if (!any) {  // integrators.py:125-127: W = 0, no engine call
      for (int i = 0; i < T.ns; ++i)
        for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) T.W[i][u] = d4(0.0);
      if (lead) {
        EikPhipmInfo inf = {};
        inf.skipped = 1;
        Wk.info[T.info_idx] = inf;
      }
      grid.sync();
      return EIK_OK;
    }
  }

  double tau0 = T.tau_init;
  int64_t m0 = T.m_init;
  if (T.slot >= 0) {
    tau0 = __ldcg(Wk.seeds + 2 * T.slot);
    m0 = (int64_t)__ldcg(Wk.seeds + 2 * T.slot + 1);
  }
  double tau;
  int64_t m;
  initial_tau_m(tau0, m0, T.rho[0], T.rho[T.ns - 1], T.m_max, n, &tau, &m);
  const int64_t m_cap = T.m_max < n ? T.m_max : n;

  const double4* y = vnz[0] ? T.v[0] : Wk.zero;
  bool y_nz = vnz[0];
  int ycur = -1;
  double t = 0.0;
  int64_t attempts = 0, acc = 0, rej = 0, mv = 0;
  const int64_t ld = Wk.m_alloc;

  for (int io = 0; io < T.ns; ++io) {
    const double t_out = T.rho[io];
    while (t < t_out) {
      ++attempts;
      if (attempts > T.max_attempts) {
        if (lead) {
          EikPhipmInfo inf = {};
          inf.substeps = acc;
          inf.rejections = rej;
          inf.matvecs = mv;
          inf.tau_final = tau;
          inf.m_final = m;
          inf.t_reached = t;
          inf.attempts = attempts - 1;
          inf.status = EIK_EPHIPM;
          Wk.info[T.info_idx] = inf;
        }
        grid.sync();
        return EIK_EPHIPM;
      }
      const double tau_nom = tau;
      const bool hits = eik_add(t, tau) >= t_out;
      if (hits) tau = eik_sub(t_out, t);

      // ---- w recurrence (phipm.py:159-182)
      const double4* wprev = y;
      bool wprev_nz = y_nz;
      double ssq = 0.0;
      for (int j = 1; j <= p; ++j) {
        double cl[MAXV];
        for (int ell = 0; ell <= p - j; ++ell) cl[ell] = pow_over_fact(t, ell);
        const bool do_mv = !(T.zero_skip && !wprev_nz);
        double4* wj = Wk.w[j];
        double r[2] = {0.0, 0.0};
        if constexpr (Op::kTiled) {
          if (do_mv) {
            ++mv;
            const double4* src = wprev;
            swe_tiled(op, [&](int64_t g, bool) { return src[g]; },
                      [&](int64_t i, double4 z, double4) {
                        double4 a = z;
                        for (int ell = 0; ell <= p - j; ++ell)
                          if (vnz[j + ell]) a = a + cl[ell] * T.v[j + ell][i];
                        wj[i] = a;
                        r[0] += nz4(a);
                        r[1] += dot4(a, a);
                      });
          }
        } else {
          if (do_mv) {
            op_pre(op, wprev, 1.0, lo, hi);
            grid.sync();
            ++mv;
          }
        }
        if (!Op::kTiled || !do_mv) {
          for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
            double4 a = do_mv ? op_main(op, wprev, u) : d4(0.0);
            for (int ell = 0; ell <= p - j; ++ell)
              if (vnz[j + ell]) a = a + cl[ell] * T.v[j + ell][u];
            wj[u] = a;
            r[0] += nz4(a);
            r[1] += dot4(a, a);
          }
        }
        grid_reduce<2>(grid, sm, r, Wk.part);
        wprev = wj;
        wprev_nz = r[0] > 0.0;
        ssq = r[1];
      }
      if (p == 0) {
        double r[2] = {0.0, 0.0};
        for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
            const double4 a = y[u];
            r[0] += nz4(a);
            r[1] += dot4(a, a);
          }
        grid_reduce<2>(grid, sm, r, Wk.part);
        wprev_nz = r[0] > 0.0;
        ssq = r[1];
      }
      const double4* wp = wprev;
      const bool wp_nz = wprev_nz;

      // ---- IOM2 Krylov decomposition (krylov.py:53-112)
      double beta = 0.0, hnext = 0.0, eps = 0.0, nh = 0.0, corner = 0.0;
      bool broke = false;
      int64_t keep = 0;
      // v_{m+1} = ((z - h1 v_{m-1}) - h2 v_m) / h_next (tiled path) or z / h_next
      const double4* vnext_z = Wk.zbuf;
      const double4* vnext_m1 = nullptr;
      const double4* vnext_v = nullptr;
      double vnext_h1 = 0.0, vnext_h2 = 0.0;
      bool vnext_expl = true;
      if (wp_nz) {
        beta = sqrt(ssq);
        const int64_t m_eff = m < n ? m : n;
        const int64_t iom = m_eff < n ? T.iom : n;
        if (blockIdx.x == 0) {
          for (int64_t q = threadIdx.x; q < m_eff * ld; q += TPB) Wk.H[q] = 0.0;
          __syncthreads();
        }
        double hcur = beta;
        const double4* raw = wp;
        keep = m_eff;
        bool tiled_done = false;
        if constexpr (Op::kTiled) {
          if (iom == 2) {
            tiled_done = true;
            // one tiled pass + one grid barrier per iteration: v_j is formed
            // on the fly from (z_{j-1}, v_{j-2}, v_{j-1}) with the previous
            // iteration's MGS coefficients, its norm taken from the Gram
            // identity (explicit pass only when that would cancel)
            double h1 = 0.0, h2 = 0.0, nm1 = 0.0;
            bool expl = false;
            for (int64_t j = 0; j < m_eff; ++j) {
              double4* vj = Wk.basis + j * NU;
              const double4* vm1 = j > 0 ? Wk.basis + (j - 1) * NU : nullptr;
              const double4* vm2 = j > 1 ? Wk.basis + (j - 2) * NU : nullptr;
              const double4* zin = (j & 1) ? Wk.zbuf : Wk.zbuf2;
              double4* zout = (j & 1) ? Wk.zbuf2 : Wk.zbuf;
              double d[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
              const double hc = hcur, a1 = h1, a2 = h2;
              const int mode = j == 0 ? 0 : (expl ? 0 : (vm2 ? 2 : 1));
              const double4* src = j == 0 ? wp : zin;
              swe_tiled(
                  op,
                  [&](int64_t g, bool own) {
                    double4 x = src[g];
                    if (mode == 2) x = x - a1 * vm2[g];
                    if (mode >= 1) x = x - a2 * vm1[g];
                    x = div4(x, hc);
                    if (own) vj[g] = x;
                    return x;
                  },
                  [&](int64_t i, double4 z, double4 x) {
                    zout[i] = z;
                    d[1] += dot4(x, z);
                    d[3] += dot4(z, z);
                    d[4] += dot4(x, x);
                    if (vm1) {
                      const double4 b = vm1[i];
                      d[0] += dot4(b, z);
                      d[2] += dot4(x, b);
                    }
                  });
              ++mv;
              if (lead) atomicAdd(Wk.kiters, 1ull);
              grid_reduce<5>(grid, sm, d, Wk.part);
              const double h1n = vm1 ? d[0] : 0.0;
              const double h2n = vm1 ? d[1] - h1n * d[2] : d[1];
              if (lead) {
                if (vm1) Wk.H[(j - 1) * ld + j] = h1n;
                Wk.H[j * ld + j] = h2n;
              }
              double hsq = d[3] - 2.0 * h2n * d[1] + h2n * h2n * d[4];
              if (vm1) hsq += -2.0 * h1n * d[0] + h1n * h1n * nm1 + 2.0 * h1n * h2n * d[2];
              expl = !(hsq > kGramSafe * d[3]);
              if (expl) {
                double r[1] = {0.0};
                for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
                  double4 z = zout[u];
                  if (vm1) z = z - h1n * vm1[u];
                  z = z - h2n * vj[u];
                  zout[u] = z;
                  r[0] += dot4(z, z);
                }
                grid_reduce<1>(grid, sm, r, Wk.part);
                hsq = r[0];
                if (lead) atomicAdd(Wk.kiters + 1, 1ull);
              }
              const double h = sqrt(hsq);
              nm1 = d[4];
              if (h < kBreakdownTol * beta) {
                broke = true;
                keep = j + 1;
                hnext = 0.0;
                break;
              }
              if (j + 1 < m_eff) {
                if (lead) Wk.H[(j + 1) * ld + j] = h;
                hcur = h;
                h1 = h1n;
                h2 = h2n;
              } else {
                hnext = h;
                vnext_z = zout;
                vnext_h1 = h1n;
                vnext_h2 = h2n;
                vnext_m1 = vm1;
                vnext_v = vj;
                vnext_expl = expl;
              }
            }
          }
        }
        for (int64_t j = 0; j < m_eff && !tiled_done; ++j) {
          double4* vj = Wk.basis + j * NU;
          const double4* vjm = j > 0 ? Wk.basis + (j - 1) * NU : nullptr;
          // v_j = raw / h (exact division), La = L v_j
          for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) vj[u] = div4(raw[u], hcur);
          op_pre(op, raw, 1.0 / hcur, lo, hi);
          grid.sync();
          // z = A v_j + projections
          double d[3] = {0.0, 0.0, 0.0};
          const bool fast = (iom == 2);
          for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
            const double4 z = op_main(op, vj, u);
            Wk.zbuf[u] = z;
            if (fast) {
              const double4 a = vj[u];
              d[1] += dot4(a, z);
              if (vjm) {
                const double4 b = vjm[u];
                d[0] += dot4(b, z);
                d[2] += dot4(a, b);
              }
            }
          }
          ++mv;
          if (lead) atomicAdd(Wk.kiters, 1ull);
          double ssz = 0.0;
          if (fast) {
            grid_reduce<3>(grid, sm, d, Wk.part);
            // MGS against v_{j-1} then v_j: <v_j, z - h1 v_{j-1}> = d1 - h1 d2
            const double h1 = d[0];
            const double h2 = vjm ? d[1] - h1 * d[2] : d[1];
            if (lead) {
              if (vjm) Wk.H[(j - 1) * ld + j] = h1;
              Wk.H[j * ld + j] = h2;
            }
            double r[1] = {0.0};
            for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
              double4 z = Wk.zbuf[u];
              if (vjm) z = z - h1 * vjm[u];
              z = z - h2 * vj[u];
              Wk.zbuf[u] = z;
              r[0] += dot4(z, z);
            }
            grid_reduce<1>(grid, sm, r, Wk.part);
            ssz = r[0];
          } else {
            // generic modified Gram-Schmidt against the last `iom` vectors
            const int64_t i0 = j - iom + 1 > 0 ? j - iom + 1 : 0;
            double cprev = 0.0;
            for (int64_t i = i0; i <= j + 1; ++i) {
              const double4* vp = i > i0 ? Wk.basis + (i - 1) * NU : nullptr;
              const double4* vi = i <= j ? Wk.basis + i * NU : nullptr;
              double r[1] = {0.0};
              for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
                double4 z = Wk.zbuf[u];
                if (vp) {
                  z = z - cprev * vp[u];
                  Wk.zbuf[u] = z;
                }
                r[0] += vi ? dot4(vi[u], z) : dot4(z, z);
              }
              grid_reduce<1>(grid, sm, r, Wk.part);
              if (i <= j) {
                cprev = r[0];
                if (lead) Wk.H[i * ld + j] = cprev;
              } else {
                ssz = r[0];
              }
            }
          }
          const double h = sqrt(ssz);
          if (h < kBreakdownTol * beta) {
            broke = true;
            keep = j + 1;
            hnext = 0.0;
            break;
          }
          if (j + 1 < m_eff) {
            // zbuf is complete: the reduction above ended with grid.sync
            if (lead) Wk.H[(j + 1) * ld + j] = h;
            hcur = h;
            raw = Wk.zbuf;
          } else {
            hnext = h;
          }
        }
        // ---- dense phi via the augmented exponential (kernels.py:148-193)
        __threadfence();
        grid.sync();
        if (blockIdx.x == 0) {
          const int dim = (int)(keep + p + 1);
          double* M0 = Wk.scr;
          for (int idx = threadIdx.x; idx < dim * dim; idx += TPB) {
            const int i = idx / dim, jj = idx - i * dim;
            double hv = 0.0;
            if (i < keep && jj < keep) hv = Wk.H[i * ld + jj];
            else if (i == 0 && jj == keep) hv = 1.0;
            else if (i >= keep && jj == i + 1 && i < keep + p) hv = 1.0;
            M0[idx] = hv;  // Hhat
          }
          __syncthreads();
          const double nrm_hat = blk_norm1(sm, M0, dim);
          for (int idx = threadIdx.x; idx < dim * dim; idx += TPB) M0[idx] = tau * M0[idx];
          __syncthreads();
          const int e = blk_expm(sm, Wk.scr, dim);
          const double* E = Wk.scr + (int64_t)e * MAXDIM * MAXDIM;
          const double tp = pow(tau, (double)p);
          const int colp = p >= 1 ? (int)keep + p - 1 : 0;
          for (int i = threadIdx.x; i < keep; i += TPB) Wk.phi[i] = E[(int64_t)i * dim + colp] / tp;
          if (threadIdx.x == 0) {
            Wk.phi[keep] = E[(int64_t)(keep - 1) * dim + keep + p];
            Wk.phi[keep + 1] = eik_mul(tau, nrm_hat);
          }
          __threadfence();
        }
        grid.sync();
        for (int i = threadIdx.x; i < keep + 2; i += TPB) sm.phi[i] = __ldcg(Wk.phi + i);
        __syncthreads();
        corner = sm.phi[keep];
        nh = sm.phi[keep + 1];
        eps = broke ? 0.0 : eik_mul(eik_mul(beta, fabs(hnext)), fabs(corner));
      }

      // ---- candidate (phipm.py:198-212, krylov.py:136-145)
      double4* cand = Wk.ybuf[ycur == 0 ? 1 : 0];
      {
        double cj[MAXV];
        for (int j = 0; j < p; ++j) cj[j] = pow_over_fact(tau, j);
        const double tp = pow(tau, (double)p);
        const double corr = (beta * hnext) * (corner / tp);
        double r[1] = {0.0};
        for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
          double4 c = d4(0.0);
          for (int j = 0; j < p; ++j) {
            const double4 wv = (j == 0) ? y[u] : Wk.w[j][u];
            c = c + cj[j] * wv;
          }
          if (wp_nz) {
            double4 s = d4(0.0);
            for (int64_t k = 0; k < keep; ++k) s = s + sm.phi[k] * Wk.basis[k * NU + u];
            double4 ap = beta * s;
            if (!broke) {
              double4 zz = vnext_z[u];
              if (!vnext_expl) {
                if (vnext_m1) zz = zz - vnext_h1 * vnext_m1[u];
                zz = zz - vnext_h2 * vnext_v[u];
              }
              ap = ap + corr * div4(zz, hnext);
            }
            c = c + tp * ap;
          }
          cand[u] = c;
          r[0] += nz4(c);
        }
        grid_reduce<1>(grid, sm, r, Wk.part);
        const bool cand_nz = r[0] > 0.0;

        // ---- controller (phipm.py:336-359)
        const double omega = eik_div(eik_mul(t_out, eps), eik_mul(tau, T.tol));
        const bool ok = omega <= T.delta;
        if (lead && Wk.trace && attempts <= Wk.trace_cap) {
          EikTraceRec tr;
          tr.attempt = attempts;
          tr.t = t;
          tr.tau = tau;
          tr.m = m;
          tr.eps_m = eps;
          tr.omega = omega;
          tr.accepted = ok ? 1 : 0;
          Wk.trace[attempts - 1] = tr;
          *Wk.trace_len = attempts;
        }
        const double tau_used = tau;
        Adapt ad = adapt_parameters(tau, m, t, eps, nh, t_out, T.rho[T.ns - 1], p,
                                    T.tol, T.delta, T.m_max, n, Wk.nnz);
        if (ok) {
          y = cand;
          ycur = ycur == 0 ? 1 : 0;
          y_nz = cand_nz;
          t = hits ? t_out : eik_add(t, tau_used);
          ++acc;
          if (hits && ad.tau < tau_nom) ad.tau = tau_nom;
        } else {
          ++rej;
        }
        tau = ad.tau > 1e-16 ? ad.tau : 1e-16;
        m = ad.m < 1 ? 1 : (ad.m > m_cap ? m_cap : ad.m);
      }
    }
    for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) T.W[io][u] = y[u];
  }
  if (lead) {
    EikPhipmInfo inf = {};
    inf.substeps = acc;
    inf.rejections = rej;
    inf.matvecs = mv;
    inf.tau_final = tau;
    inf.m_final = m;
    inf.t_reached = t;
    inf.attempts = attempts;
    inf.status = EIK_OK;
    Wk.info[T.info_idx] = inf;
    if (T.slot >= 0) {
      Wk.seeds[2 * T.slot] = tau;
      Wk.seeds[2 * T.slot + 1] = (double)m;
    }
  }
  __threadfence();
  grid.sync();
  return EIK_OK;
}

}  // namespace eik
