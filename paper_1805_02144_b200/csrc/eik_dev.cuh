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

#ifndef EIK_TPB
#define EIK_TPB 256
#endif
#ifndef EIK_MINB
#define EIK_MINB 2
#endif
constexpr int TPB = EIK_TPB;    // threads per CTA
constexpr int MINB = EIK_MINB;  // co-resident CTAs per SM (register budget)
constexpr int NWARP = TPB / 32;
constexpr int NPART = 8;   // doubles per CTA partial record
constexpr int MAXV = 8;    // v_0..v_7
constexpr int MAXNS = 8;   // output points
constexpr int MAXDIM = kDenseCap;
constexpr int KMAX = 8;    // stencil slots per cell (self + up to 7)
constexpr int KCMAX = 6;   // off-diagonal slots of the compact stencil (hexagons)
constexpr int NOPS = 10;
// Gram-identity norm of the orthogonalised vector is used while it keeps
// h^2 > kGramSafe ||z||^2 (relative error of h below ~1e-14); else an
// explicit orthogonalisation pass recomputes it.
constexpr double kGramSafe = 1e-2;   // Gx Gy Gz Dx Dy Dz Vx Vy Vz L
enum { OP_GX = 0, OP_GY, OP_GZ, OP_DX, OP_DY, OP_DZ, OP_VX, OP_VY, OP_VZ, OP_L };

// ------------------------------------------------------------ profiling
// EIK_PROF builds: CTA 0 / thread 0 accumulates clock64() deltas per phase
// category (read back with eik_prof_read); zero cost otherwise.
enum { PC_RHS = 0, PC_NNZ, PC_WREC, PC_KRYLOV, PC_DENSE, PC_CAND, PC_DEV, PC_MISC, PC_N = 16 };
__device__ unsigned long long g_prof[PC_N];
struct ProfClock {
#if EIK_PROF && defined(__CUDA_ARCH__)
  long long t;
  __device__ ProfClock() : t(clock64()) {}
  __device__ void mark(int k) {
    const long long n = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) g_prof[k] += (unsigned long long)(n - t);
    t = n;
  }
  __device__ void skip() { t = clock64(); }
#else
  __device__ void mark(int) {}
  __device__ void skip() {}
#endif
};

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

// 256-bit global accesses (one LDG/STG.E.ENL2.256 per cell instead of two
// 128-bit halves hitting the same sector twice).  ldv: coherent (data written
// earlier in the same kernel, ordered by a barrier); ldv_nc: read-only for the
// kernel's lifetime.
__device__ __forceinline__ double4 ldv(const double4* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double4 ldv_nc(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldv2_nc(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void stv(double4* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
               "d"(v.w)
               : "memory");
}

// L2 residency hints (EIK_L2POL): the Krylov vectors written by a pass are
// stored evict_last (read again in the next iteration, first by the tiles
// that wrote them last, see Form::rev); the coefficient stream is loaded
// evict_first.
#ifndef EIK_L2POL
#define EIK_L2POL 1
#endif

__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void stv_pol(double4* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v.x),
               "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ double ld_stream_pol(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---------------------------------------------------------------- shared
constexpr int SMW = 16;  // tiles of metadata staged at a time
struct Smem {
  double red[NWARP][NPART];
  double tot[NPART];
  double phi[MAXDIM + 4];
  int ival[4];
  int par;      // partial-buffer parity (double buffering, see grid_reduce)
  int meta[SMW][7];  // tiled pass: metadata of the CTA's next SMW tiles
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

// Deterministic grid-wide sums: every CTA writes its partials, value-major
// (part[k][b], k < NV, rows padded to a multiple of 32 CTAs), and after the
// grid barrier every CTA reduces them in the same fixed order -- warp k sums
// value k with coalesced loads -- so all CTAs hold bit-identical totals.
// Partials are double-buffered: a fast CTA may start the next reduction's
// store while a slow CTA still reads this one's; the two buffers alternate
// and at least one grid.sync separates reuse.  `part` holds 2 * NPART * Gp
// doubles, Gp = gridDim.x rounded up to 32.
__host__ __device__ constexpr int part_stride(int G) { return (G + 31) & ~31; }

template <int NV>
__device__ void grid_reduce(cg::grid_group& grid, Smem& sm, double (&v)[NV], double* part) {
  static_assert(NV <= NPART && NV <= TPB, "partials per CTA");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = gridDim.x, Gp = part_stride(G);
  const int par = sm.par;
  double* P = part + (int64_t)par * NPART * Gp;
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
    __stcg(P + (int64_t)threadIdx.x * Gp + blockIdx.x, s);
  }
  if (threadIdx.x == 0) sm.par = par ^ 1;
  grid.sync();
  // one warp per reduced value (round robin when a CTA has fewer warps)
  for (int k = w; k < NV; k += NWARP) {
    const double* row = P + (int64_t)k * Gp;
    double s = 0.0;
    for (int b0 = 0; b0 < G; b0 += 32 * 8) {
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int b = b0 + lane + 32 * q;
        x[q] = b < G ? __ldcg(row + b) : 0.0;
      }
      s += ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]));
    }
    s = warp_sum(s);
    if (lane == 0) sm.tot[k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sm.tot[k];
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
  double4* gn;           // g_n = F*(u_n) - J* u_n (tiled D(U), see DevStep)
  double scale;          // A x = scale * (J x)   (integrators.py:117)
  // n_A counting data
  const double* df1;     // [K][N] Df(i, slot) (0 where Df has no entry)
  const int* dfx;        // [N] nonzero Df entries outside the slot set
  const int* cnt;        // [N] valid slots
  // tiled single-pass Krylov iteration (tiles = contiguous ranges of the device cell order;
  // each tile's 2-ring halo is staged in shared memory)
  int ntiles;
  const int* t_cell0;    // first own cell
  const int* t_nT;       // own cells (<= TPB)
  const int* t_nE1;      // own + 1-ring halo
  const int* t_nE2;      // own + 1-ring + 2-ring halo
  const int* t_e2off;    // offset into e2map
  const int* t_e1off;    // offset into lnbr (rows)
  const int* e2map;      // local -> global cell id, order [own, H1, H2]
  const short* lnbr;     // [rows][8] local off-diagonal neighbours of E1 cells
  const double* coefc;   // off-diagonal G, D, V (compact stencil), 54 runs (slot-major) per
                         // tile: tile-major blocks [tile][54][TILE] at t_coff * 16
                         // (tilecoef; run stride pad16(nT) without EIK_FIXCS), or the
                         // global runs [54][NC]
  int64_t NC;            // global run stride (N rounded up to even)
  const int* t_coff;     // per tile: block offset / 16 doubles (0 for global runs)
  int tilecoef;
  const double* Lc;      // [N][8] off-diagonal Laplacian row (cell-major)
  const double* LcE1;    // [sum of tile E1][6] Laplacian rows of every tile's E1 cells
                         // in local order (offset t_e1off * 6)
  int KC;                // off-diagonal slots
  int tiled_ok;          // compact stencil valid for this operator set
  unsigned long long* prof;  // EIK_PROF builds: per-step cycle counters
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
// The tiled Krylov pass works on the compact ("difference form") stencil:
// for operators whose diagonal is minus (G, V, L) or plus (D) the sum of
// the row's off-diagonal entries -- true for the sphere grid and for the
// reference's planar operators -- only the off-diagonal slots are stored and
//   (G e)_i = sum_j G_ij (e_j - e_i),  (D f)_i = sum_j D_ij (f_j + f_i).
//
// Tiles are contiguous ranges of <= TPB device cells (compact patches, see
// the device cell order in eik_swe_create); a CTA stages a tile's input
// vector on the tile's 2-ring halo E2 in shared memory and every thread runs
// the three steps of the tile in turn (256-thread CTAs, 2 per SM).
//
// Shared memory is kept small on purpose: it is carved out of the same
// 256 KB per SM as the L1 that holds the pass's in-flight global loads.
// Measured at L8 (us per Krylov iteration): +40 KB of shared memory per CTA
// 159 vs 117; TMA / cp.async staging of the per-tile static data or of the
// coefficient stream 157-171; L2 prefetch of the coefficient runs 125-139.
#ifndef EIK_PROF
#define EIK_PROF 0
#endif
constexpr int TILE = TPB;          // max own cells per tile
constexpr int NCOEF = KCMAX * 9;   // compact G/D/V runs per cell (slot-major)

#ifndef EIK_SPLIT
#define EIK_SPLIT 1
#endif
// A double4 array in shared memory.  With EIK_SPLIT the (x,y) and (z,w)
// halves live in two double2 arrays: a warp's random 16-byte reads then
// spread over all 8 bank groups instead of the 4 a 32-byte stride allows.
struct SArr {
  double2* p;
  int n;
};
__device__ __forceinline__ double4 sld(const SArr& a, int l) {
#if EIK_SPLIT
  const double2 u = a.p[l], v = a.p[a.n + l];
  return make_double4(u.x, u.y, v.x, v.y);
#else
  return reinterpret_cast<const double4*>(a.p)[l];
#endif
}
__device__ __forceinline__ void sst(const SArr& a, int l, double4 v) {
#if EIK_SPLIT
  a.p[l] = make_double2(v.x, v.y);
  a.p[a.n + l] = make_double2(v.z, v.w);
#else
  reinterpret_cast<double4*>(a.p)[l] = v;
#endif
}

struct TileSmem {
  SArr x;   // [e2max] input vector on E2
  SArr La;  // [e1max] L x on E1
  SArr U;   // [e1max] linearisation state on E1
};
__host__ __device__ constexpr size_t tile_smem_bytes(int e1max, int e2max) {
  return 128 + (size_t)e2max * 32 + (size_t)e1max * 64;
}
__device__ __forceinline__ TileSmem tile_smem(const SweOp& S) {
  extern __shared__ __align__(128) unsigned char dsm[];
  TileSmem t;
  double2* q = reinterpret_cast<double2*>(dsm + 128);
  t.x = SArr{q, S.e2max};
  q += 2 * S.e2max;
  t.La = SArr{q, S.e1max};
  q += 2 * S.e1max;
  t.U = SArr{q, S.e1max};
  return t;
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
// the 6 off-diagonal Laplacian coefficients of one E1 row (16-byte loads)
struct Lrow {
  double v[8];
};
__device__ __forceinline__ Lrow load_lrow(const double* p) {
  const double2 a = ldv2_nc(p), b = ldv2_nc(p + 2), c = ldv2_nc(p + 4);
  return Lrow{{a.x, a.y, b.x, b.y, c.x, c.y, 0.0, 0.0}};
}

// compact coefficient order in coefc: [KCMAX][9][NC], ops Vx Vy Vz Gx Gy Gz Dx Dy Dz.
struct JvAcc {
  double zeta, gx, gy, gz, dv, l0, l1, l2, l3;
};

#ifndef EIK_CHUNK
#define EIK_CHUNK 3
#endif
#ifndef EIK_EXP_HALFDV
#define EIK_EXP_HALFDV 0
#endif
// EIK_SMETA: tile metadata staged in shared memory 16 tiles at a time;
// EIK_PFM (with it): the next tile's halo map prefetched into L1 during step 3
#ifndef EIK_SMETA
#define EIK_SMETA 1
#endif
#ifndef EIK_PFM
#define EIK_PFM 1
#endif
// unroll factor of the candidate's sum over the basis vectors (loads in flight)
#ifndef EIK_CANDU
#define EIK_CANDU 4
#endif
constexpr int kCandU = EIK_CANDU;
// EIK_SHDIV: form_x divides by h through a shared reciprocal (see there)
#ifndef EIK_SHDIV
#define EIK_SHDIV 1
#endif
// EIK_ROW0: every thread loads row threadIdx.x of the tile's step-2 rows
// before the barrier that ends step 1 and keeps it for step 3 (own cells)
#ifndef EIK_ROW0
#define EIK_ROW0 0
#endif
// EIK_PF5: L2 prefetch of step 3's first coefficient chunk just before the
// barrier that ends step 2
#ifndef EIK_PF5
#define EIK_PF5 1
#endif
// runs [0, EIK_PF5A) are prefetched at the start of step 2, runs
// [EIK_PF5A, EIK_PF5A + EIK_PF5N) at its end (27 runs = the first chunk)
#ifndef EIK_PF5A
#define EIK_PF5A 0
#endif
#ifndef EIK_PF5N
#define EIK_PF5N 27
#endif
// EIK_BAR1: the barrier that ends a tile is taken inside the next tile's
// step 1, after its gathers are issued and before its first shared-memory
// store (a warp that finishes step 3 early starts the next tile's gathers)
#ifndef EIK_BAR1
#define EIK_BAR1 1
#endif
// One chunk of CH slots' G/D/V coefficients of own cell i (9 per slot).
template <int CH>
struct CoefChunk {
  double v[CH][9];
};
// cptr: the cell's entry of run 0, cs: run stride (doubles)
// EIK_FIXCS (default): every tile block has run stride TILE, so the 54 loads
// of a cell are one base register plus immediate offsets (no per-load address
// arithmetic); 0 keeps the run stride a run-time value (pad16(nT) blocks, or
// the global runs with EIK_TILECOEF=0 in the environment)
#ifndef EIK_FIXCS
#define EIK_FIXCS 1
#endif
#if EIK_FIXCS
struct CoefPtr {
  const double* p;
  static constexpr int64_t cs = TPB;
  __device__ __forceinline__ CoefPtr(const double* q, int64_t) : p(q) {}
};
#else
struct CoefPtr {
  const double* p;
  int64_t cs;
};
#endif
template <int CH>
__device__ __forceinline__ void coef_load(const CoefPtr& C, int s0, CoefChunk<CH>& cf) {
  const int64_t st = (int64_t)9 * C.cs;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const double* cp = C.p + (s0 + k) * st;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
#if EIK_EXP_HALFDV
      // experiment only: D not streamed (V reused) -- wrong results
      if (q >= 6) { cf.v[k][q] = cf.v[k][q - 6]; continue; }
#endif
#if EIK_L2POL
      cf.v[k][q] = ld_stream_pol(cp + q * C.cs, pol_evict_first());
#else
      cf.v[k][q] = __ldcs(cp + q * C.cs);
#endif
    }
  }
}
// own-cell terms shared by every slot
struct JvOwn {
  double4 ai, Ui, lai;
  double ei, fxi, fyi, fzi;
};
__device__ __forceinline__ JvOwn jv_own(const SweOp& S, double4 ai, double4 Ui, double4 lai) {
  JvOwn o;
  o.ai = ai;
  o.Ui = Ui;
  o.lai = lai;
  o.ei = Ui.x * ai.x + Ui.y * ai.y + Ui.z * ai.z + S.g * ai.w;
  o.fxi = Ui.w * ai.x + Ui.x * ai.w;
  o.fyi = Ui.w * ai.y + Ui.y * ai.w;
  o.fzi = Ui.w * ai.z + Ui.z * ai.w;
  return o;
}
// accumulate slots [s0, s0+CH) with their coefficients in cf
template <int CH>
__device__ __forceinline__ void jv_accum(const SweOp& S, const TileSmem& ts, const short* row,
                                         const double* lc, int s0, const CoefChunk<CH>& cf,
                                         const JvOwn& o, JvAcc& a) {
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int s = s0 + k;
    const int l = row[s];
    const double vx = cf.v[k][0], vy = cf.v[k][1], vz = cf.v[k][2];
    const double gcx = cf.v[k][3], gcy = cf.v[k][4], gcz = cf.v[k][5];
    const double dx = cf.v[k][6], dy = cf.v[k][7], dz = cf.v[k][8];
    const double l0 = lc[s];
    const double4 aj = sld(ts.x, l);
    const double4 U = sld(ts.U, l);
    const double4 la = sld(ts.La, l);
    a.zeta += vx * (aj.x - o.ai.x) + vy * (aj.y - o.ai.y) + vz * (aj.z - o.ai.z);
    const double e = U.x * aj.x + U.y * aj.y + U.z * aj.z + S.g * aj.w;
    a.gx += gcx * (e - o.ei);
    a.gy += gcy * (e - o.ei);
    a.gz += gcz * (e - o.ei);
    a.dv += dx * ((U.w * aj.x + U.x * aj.w) + o.fxi) + dy * ((U.w * aj.y + U.y * aj.w) + o.fyi) +
            dz * ((U.w * aj.z + U.z * aj.w) + o.fzi);
    a.l0 += l0 * (la.x - o.lai.x);
    a.l1 += l0 * (la.y - o.lai.y);
    a.l2 += l0 * (la.z - o.lai.z);
    a.l3 += l0 * (la.w - o.lai.w);
  }
}

// Sum over all KCMAX slots of own cell i (x, La, U in smem).  Slots are
// processed in chunks of EIK_CHUNK: all 9*CHUNK coefficient loads of a chunk
// are issued before any of them is used (a compiler memory fence keeps them
// together), so each thread keeps ~27 streaming loads in flight instead of
// the handful the default schedule interleaves with the math.
constexpr int JCH = (EIK_CHUNK < KCMAX) ? EIK_CHUNK : KCMAX;
using JvChunk = CoefChunk<JCH>;
__device__ __forceinline__ JvAcc swe_jv_sum(const SweOp& S, const TileSmem& ts, const short* row,
                                            const double* lc, const CoefPtr& C, double4 ai,
                                            double4 Ui, double4 lai) {
  const JvOwn o = jv_own(S, ai, Ui, lai);
  JvAcc a = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  constexpr int CH = JCH;
#pragma unroll
  for (int k0 = 0; k0 < KCMAX; k0 += CH) {
    CoefChunk<CH> cf;
    coef_load<CH>(C, k0, cf);
    asm volatile("" ::: "memory");
    jv_accum<CH>(S, ts, row, lc, k0, cf, o, a);
  }
  return a;
}


__device__ __forceinline__ double4 swe_jv_finish(const SweOp& S, const JvAcc& a, double4 q,
                                                 double4 ai, double4 Ui) {
  const double px = q.y * Ui.z - q.z * Ui.y;
  const double py = q.z * Ui.x - q.x * Ui.z;
  const double pz = q.x * Ui.y - q.y * Ui.x;
  const double cx = q.y * ai.z - q.z * ai.y;
  const double cy = q.z * ai.x - q.x * ai.z;
  const double cz = q.x * ai.y - q.y * ai.x;
  double4 r;
  r.x = -(px * a.zeta) - q.w * cx - a.gx - S.nu * a.l0;
  r.y = -(py * a.zeta) - q.w * cy - a.gy - S.nu * a.l1;
  r.z = -(pz * a.zeta) - q.w * cz - a.gz - S.nu * a.l2;
  r.w = -a.dv - S.nu * a.l3;
  return r;
}

// Step-3 operators of the tiled pass (own cell i, its staged values ai,
// Ui (the E1 stage) and lai = (L x)_i):
//   JvStep:  z = scale * (J x)_i, E1 stage = linearisation state U;
//   RhsStep: F(w)_i (swe.py:149-168) on the compact stencil, w staged as x,
//            E1 stage = (h_s, 0, 0, 0).
struct JvStep {
  static constexpr bool kStageHs = false;
  static constexpr bool kE1Only = false;
  __device__ __forceinline__ double4 operator()(const SweOp& S, const TileSmem& ts,
                                                const short* row, const double* lc, int64_t i,
                                                const CoefPtr& C, double4 ai, double4 Ui,
                                                double4 lai) const {
    const JvAcc a = swe_jv_sum(S, ts, row, lc, C, ai, Ui, lai);
    return S.scale * swe_jv_finish(S, a, ldv(S.ne + i), ai, Ui);
  }
};

// F on the compact stencil, with the G E sum split into its h_s-free part
// (gx..) and the h_s part (hx..), and, for the step start, the J* sum of
// J* u at u itself (jx..: e_j = u_j . u_j + g h_j).  * = without Df and h_s.
struct RhsAcc {
  double zeta, gx, gy, gz, hx, hy, hz, jx, jy, jz, dv, l0, l1, l2, l3;
};
template <int CH>
__device__ __forceinline__ void rhs_accum(const SweOp& S, const TileSmem& ts, const short* row,
                                          const double* lc, int s0, const CoefChunk<CH>& cf,
                                          double4 wi, double Ei, double Hi, double Ji,
                                          double4 lai, RhsAcc& a) {
  const double fxi = wi.x * wi.w, fyi = wi.y * wi.w, fzi = wi.z * wi.w;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int s = s0 + k;
    const int l = row[s];
    const double vx = cf.v[k][0], vy = cf.v[k][1], vz = cf.v[k][2];
    const double gcx = cf.v[k][3], gcy = cf.v[k][4], gcz = cf.v[k][5];
    const double dx = cf.v[k][6], dy = cf.v[k][7], dz = cf.v[k][8];
    const double l0 = lc[s];
    const double4 wj = sld(ts.x, l);
    const double hsj = sld(ts.U, l).x;
    const double4 la = sld(ts.La, l);
    a.zeta += vx * (wj.x - wi.x) + vy * (wj.y - wi.y) + vz * (wj.z - wi.z);
    const double Ej = 0.5 * (wj.x * wj.x + wj.y * wj.y + wj.z * wj.z) + S.g * wj.w;
    a.gx += gcx * (Ej - Ei);
    a.gy += gcy * (Ej - Ei);
    a.gz += gcz * (Ej - Ei);
    const double Hj = S.g * hsj;
    a.hx += gcx * (Hj - Hi);
    a.hy += gcy * (Hj - Hi);
    a.hz += gcz * (Hj - Hi);
    const double Jj = (wj.x * wj.x + wj.y * wj.y + wj.z * wj.z) + S.g * wj.w;
    a.jx += gcx * (Jj - Ji);
    a.jy += gcy * (Jj - Ji);
    a.jz += gcz * (Jj - Ji);
    a.dv += dx * (wj.x * wj.w + fxi) + dy * (wj.y * wj.w + fyi) + dz * (wj.z * wj.w + fzi);
    a.l0 += l0 * (la.x - lai.x);
    a.l1 += l0 * (la.y - lai.y);
    a.l2 += l0 * (la.z - lai.z);
    a.l3 += l0 * (la.w - lai.w);
  }
}

struct RhsStep {
  static constexpr bool kStageHs = true;
  static constexpr bool kE1Only = false;
  bool write_ne;  // store (n, eta) of every own cell to S.ne (linearisation at w)
  bool write_gn;  // store g_n = F*(w) - J*(w) w to S.gn (for DevStep)
  __device__ __forceinline__ double4 operator()(const SweOp& S, const TileSmem& ts,
                                                const short* row, const double* lc, int64_t i,
                                                const CoefPtr& C, double4 wi, double4 hsi4,
                                                double4 lai) const {
    const double Ei = 0.5 * (wi.x * wi.x + wi.y * wi.y + wi.z * wi.z) + S.g * wi.w;
    const double Hi = S.g * hsi4.x;
    const double Ji = (wi.x * wi.x + wi.y * wi.y + wi.z * wi.z) + S.g * wi.w;
    RhsAcc a = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    constexpr int CH = (EIK_CHUNK < KCMAX) ? EIK_CHUNK : KCMAX;
#pragma unroll
    for (int k0 = 0; k0 < KCMAX; k0 += CH) {
      CoefChunk<CH> cf;
      coef_load<CH>(C, k0, cf);
      asm volatile("" ::: "memory");
      rhs_accum<CH>(S, ts, row, lc, k0, cf, wi, Ei, Hi, Ji, lai, a);
    }
    const double4 q = S.nf[i];
    const double eta = a.zeta + q.w;
    if (write_ne) S.ne[i] = make_double4(q.x, q.y, q.z, eta);
    const double px = q.y * wi.z - q.z * wi.y;
    const double py = q.z * wi.x - q.x * wi.z;
    const double pz = q.x * wi.y - q.y * wi.x;
    if (write_gn) {
      // F*(w) - J*(w) w, the same expression shapes as DevStep
      double4 fs, js;
      fs.x = -eta * px - a.gx;
      fs.y = -eta * py - a.gy;
      fs.z = -eta * pz - a.gz;
      fs.w = -a.dv;
      js.x = -(px * a.zeta) - eta * px - a.jx;
      js.y = -(py * a.zeta) - eta * py - a.jy;
      js.z = -(pz * a.zeta) - eta * pz - a.jz;
      js.w = -(2.0 * a.dv);
      S.gn[i] = fs - js;
    }
    double4 r;
    r.x = -eta * px - (a.gx + a.hx) - S.nu * a.l0;
    r.y = -eta * py - (a.gy + a.hy) - S.nu * a.l1;
    r.z = -eta * pz - (a.gz + a.hz) - S.nu * a.l2;
    r.w = -a.dv - S.nu * a.l3;
    return r;
  }
};

// D(U) = F(U) - f_n - J_n (U - u_n)  (integrators.py:101-102) in one 1-ring
// pass: Df and the h_s term of F are linear in U and cancel exactly, and J is
// linear, so D(U) = [F*(U) - J*_n U] - g_n with g_n = F*(u_n) - J*_n u_n
// (RhsStep at the step start), * = without Df and h_s.  Staged: U as x and
// the linearisation state u_n on E1; no Laplacian step.
struct DevStep {
  static constexpr bool kStageHs = false;
  static constexpr bool kE1Only = true;
  __device__ __forceinline__ double4 operator()(const SweOp& S, const TileSmem& ts,
                                                const short* row, const double* /*lc*/,
                                                int64_t i, const CoefPtr& C, double4 Ui,
                                                double4 li, double4 /*lai*/) const {
    const double Ei = 0.5 * (Ui.x * Ui.x + Ui.y * Ui.y + Ui.z * Ui.z) + S.g * Ui.w;
    const double ei = li.x * Ui.x + li.y * Ui.y + li.z * Ui.z + S.g * Ui.w;
    const double fxi = Ui.x * Ui.w, fyi = Ui.y * Ui.w, fzi = Ui.z * Ui.w;
    const double kxi = li.w * Ui.x + li.x * Ui.w, kyi = li.w * Ui.y + li.y * Ui.w,
                 kzi = li.w * Ui.z + li.z * Ui.w;
    double zeta = 0.0, gx = 0.0, gy = 0.0, gz = 0.0, jx = 0.0, jy = 0.0, jz = 0.0, dv = 0.0,
           dj = 0.0;
    constexpr int CH = (EIK_CHUNK < KCMAX) ? EIK_CHUNK : KCMAX;
#pragma unroll
    for (int k0 = 0; k0 < KCMAX; k0 += CH) {
      CoefChunk<CH> cf;
      coef_load<CH>(C, k0, cf);
      asm volatile("" ::: "memory");
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int l = row[k0 + k];
        const double vx = cf.v[k][0], vy = cf.v[k][1], vz = cf.v[k][2];
        const double gcx = cf.v[k][3], gcy = cf.v[k][4], gcz = cf.v[k][5];
        const double dx = cf.v[k][6], dy = cf.v[k][7], dz = cf.v[k][8];
        const double4 Uj = sld(ts.x, l);
        const double4 lj = sld(ts.U, l);
        zeta += vx * (Uj.x - Ui.x) + vy * (Uj.y - Ui.y) + vz * (Uj.z - Ui.z);
        const double Ej = 0.5 * (Uj.x * Uj.x + Uj.y * Uj.y + Uj.z * Uj.z) + S.g * Uj.w;
        gx += gcx * (Ej - Ei);
        gy += gcy * (Ej - Ei);
        gz += gcz * (Ej - Ei);
        const double ej = lj.x * Uj.x + lj.y * Uj.y + lj.z * Uj.z + S.g * Uj.w;
        jx += gcx * (ej - ei);
        jy += gcy * (ej - ei);
        jz += gcz * (ej - ei);
        dv += dx * (Uj.x * Uj.w + fxi) + dy * (Uj.y * Uj.w + fyi) + dz * (Uj.z * Uj.w + fzi);
        dj += dx * ((lj.w * Uj.x + lj.x * Uj.w) + kxi) + dy * ((lj.w * Uj.y + lj.y * Uj.w) + kyi) +
              dz * ((lj.w * Uj.z + lj.z * Uj.w) + kzi);
      }
    }
    const double4 q = ldv(S.ne + i);  // (n, eta_n)
    const double f = S.nf[i].w;
    const double etaU = zeta + f;
    const double px = q.y * Ui.z - q.z * Ui.y;  // n x U  (also P of F at U)
    const double py = q.z * Ui.x - q.x * Ui.z;
    const double pz = q.x * Ui.y - q.y * Ui.x;
    const double nx = q.y * li.z - q.z * li.y;  // n x u_n (P of J)
    const double ny = q.z * li.x - q.x * li.z;
    const double nz = q.x * li.y - q.y * li.x;
    double4 fs, js;
    fs.x = -etaU * px - gx;
    fs.y = -etaU * py - gy;
    fs.z = -etaU * pz - gz;
    fs.w = -dv;
    js.x = -(nx * zeta) - q.w * px - jx;
    js.y = -(ny * zeta) - q.w * py - jy;
    js.z = -(nz * zeta) - q.w * pz - jz;
    js.w = -dj;
    return (fs - js) - S.gn[i];
  }
};

// How a tiled pass builds its input vector on the fly at every E2 cell:
//   x = ((src - a1 * vm2) - a2 * vm1) / h     (vm2 / vm1 optional)
// i.e. the MGS update and normalisation of krylov.py:91-104 fused into the
// load; own cells also store x (the new basis vector) to `out`.
struct Form {
  const double4* src;
  const double4* vm2;
  const double4* vm1;
  double a1, a2, h;
  double4* out;
  const double4* epi_vm1;  // own-cell vector handed to the epilogue (may be null)
  int rev = 0;             // walk the CTA's tiles in reverse order
};
#ifndef EIK_REV
#define EIK_REV 1
#endif
// EIK_PF2: prefetch the tile's step-2 rows (E1 neighbour rows + Laplacian
// rows) into L1 at the start of step 1; EIK_PFT: load the next tile's
// metadata and prefetch its halo map during step 3 of the current tile
#ifndef EIK_PF2
#define EIK_PF2 1
#endif
// EIK_PF4: at the start of step 2, prefetch into L1 the own cells' runs that
// step 3 reads last: (n, eta) and the epilogue's v_{j-1}
#ifndef EIK_PF4
#define EIK_PF4 1
#endif
#ifndef EIK_PFT
#define EIK_PFT 0
#endif

__device__ __forceinline__ double4 form_x(const Form& f, double4 s0, double4 s1,
                                          double4 s2) {
  double4 x = s0;
  if (f.vm2) x = x - f.a1 * s1;
  if (f.vm1) x = x - f.a2 * s2;
#if EIK_SHDIV
  // x / h for the four components with one shared reciprocal (the tiled pass
  // forms two halo cells per thread: 8 divisions by the same h): r = RN(1 / h),
  // q0 = RN(x r), q = RN(q0 + (x - q0 h) r) with the remainder exact by FMA --
  // the correctly rounded quotient (Markstein), i.e. the same bits as x / h
  // unless h's significand is all ones (tests/host/shared_div.c compares the
  // two on 2e7 random pairs)
  const double r = 1.0 / f.h;
  auto dv = [&](double a) {
    const double q0 = a * r;
    return fma(fma(-q0, f.h, a), r, q0);
  };
  return make_double4(dv(x.x), dv(x.y), dv(x.z), dv(x.w));
#else
  return div4(x, f.h);
#endif
}

// this CTA's tiles are t = blockIdx.x + k * gridDim.x, k < tile_count; rev walks
// them backwards (alternate Krylov iterations: the tiles written last in one
// iteration are read first in the next, while their vectors are in L2)
__device__ __forceinline__ int tile_count(const SweOp& S) {
  return S.ntiles > (int)blockIdx.x ? (S.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
}
__device__ __forceinline__ int tile_index(int k, int kt, int rev) {
  return (int)blockIdx.x + (EIK_REV && rev ? kt - 1 - k : k) * (int)gridDim.x;
}
// metadata of tiles [k, k + SMW) of the walk into sm.meta (one thread per tile)
__device__ __forceinline__ void tile_meta_fill(Smem& sm, const SweOp& S, int k, int kt, int rev) {
  if ((int)threadIdx.x < SMW && k + (int)threadIdx.x < kt) {
    const int tt = tile_index(k + threadIdx.x, kt, rev);
    int* m = sm.meta[threadIdx.x];
    m[0] = __ldg(S.t_cell0 + tt);
    m[1] = __ldg(S.t_nT + tt);
    m[2] = __ldg(S.t_nE1 + tt);
    m[3] = __ldg(S.t_nE2 + tt);
    m[4] = __ldg(S.t_e2off + tt);
    m[5] = __ldg(S.t_e1off + tt);
    m[6] = __ldg(S.t_coff + tt);
  }
}
// One pass over every tile: x on E2 -> smem, L x on E1, z = scale * J x on
// the own cells -> epi(i, z, x_i, epi_vm1_i).  A whole Krylov iteration
// (orthogonalise + normalise v_j, L v_j, J v_j, projections) is one such
// pass: one HBM sweep and one grid barrier per iteration.
template <class Step, class Epi>
__device__ void swe_tiled_op(Smem& sm, const SweOp& S, const Form& F, const Step& step,
                             const Epi& epi) {
  const TileSmem ts = tile_smem(S);
#if EIK_PROF
  long long pst[3] = {0, 0, 0}, pt = clock64();
#define SRP_MARK(k) { const long long n_ = clock64(); pst[k] += n_ - pt; pt = n_; }
#else
#define SRP_MARK(k)
#endif
  const int kt = tile_count(S);
  auto tile_of = [&](int k) { return tile_index(k, kt, F.rev); };
  struct TileMeta {
    int64_t c0;
    int nT, nE1, nE2, e2off, e1off, coff;
  };
  auto load_meta = [&](int t) {
    TileMeta m;
    m.c0 = __ldg(S.t_cell0 + t);
    m.nT = __ldg(S.t_nT + t);
    m.nE1 = __ldg(S.t_nE1 + t);
    m.nE2 = __ldg(S.t_nE2 + t);
    m.e2off = __ldg(S.t_e2off + t);
    m.e1off = __ldg(S.t_e1off + t);
    m.coff = __ldg(S.t_coff + t);
    return m;
  };
  TileMeta nxt;
  if (EIK_PFT && kt > 0) nxt = load_meta(tile_of(0));
#if EIK_SMETA
  // the metadata of this CTA's next SMW tiles, staged in shared memory by one
  // thread per tile (one round trip per SMW tiles instead of one per tile)
  auto smeta = [&](int k) {
    const int* m = sm.meta[k % SMW];
    return TileMeta{m[0], m[1], m[2], m[3], m[4], m[5], m[6]};
  };
#endif
  for (int k = 0; k < kt; ++k) {
    const int t = tile_of(k);
#if EIK_SMETA
    if (k % SMW == 0) {
      if (k) __syncthreads();  // every warp has read the previous window
      tile_meta_fill(sm, S, k, kt, F.rev);
      __syncthreads();
    }
    const TileMeta cur = smeta(k);
#else
    const TileMeta cur = EIK_PFT ? nxt : load_meta(t);
#endif
    const int64_t c0 = cur.c0;
    const int nT = cur.nT, nE1 = cur.nE1, nE2 = cur.nE2;
    if (nT == 0) {  // uniform over the CTA
      if (EIK_PFT && k + 1 < kt) nxt = load_meta(tile_of(k + 1));
      continue;
    }
    const int* map = S.e2map + cur.e2off;
    const int e1off = cur.e1off;
    const short* rows = S.lnbr + (int64_t)e1off * 8;
    const double* lce1 = S.LcE1 + (int64_t)e1off * 6;
    // the tile's 54 coefficient runs: entry of own cell c at ctile + c, run stride cstr
    const double* ctile = S.tilecoef ? S.coefc + (int64_t)cur.coff * 16 : S.coefc + c0;
#if EIK_FIXCS
    constexpr int64_t cstr = TPB;
#else
    const int64_t cstr = S.tilecoef ? (int64_t)((nT + 15) & ~15) : S.NC;
#endif
    if (EIK_PF2 && !Step::kE1Only) {
      // step-2 rows of this tile: nE1 x 16 B (rows) + nE1 x 48 B (Laplacian)
      const int l1 = (nE1 * 16 + 127) >> 7, l2 = (nE1 * 48 + 127) >> 7;
      auto pf = [&](int q) {
        prefetch_l1(q < l1 ? (const char*)rows + ((int64_t)q << 7)
                           : (const char*)lce1 + ((int64_t)(q - l1) << 7));
      };
      // one line per thread covers a tile of up to TPB cells (no loop in the common case)
      if ((int)threadIdx.x < l1 + l2) pf(threadIdx.x);
      if (l1 + l2 > TPB)
        for (int q = threadIdx.x + TPB; q < l1 + l2; q += TPB) pf(q);
    }
    // step 1: x on E2 (two cells per thread per round, all loads issued first)
    const int nEs = Step::kE1Only ? nE1 : nE2;  // cells staged in step 1
    for (int base = 0; base < nEs; base += 2 * TPB) {
      const int ca = base + threadIdx.x, cb = ca + TPB;
      const bool va = ca < nEs, vb = cb < nEs;
      const int ga = va ? __ldg(map + ca) : 0;
      const int gb = vb ? __ldg(map + cb) : 0;
      double4 a0 = d4(0.0), a1 = d4(0.0), a2 = d4(0.0), b0 = d4(0.0), b1 = d4(0.0),
              b2 = d4(0.0), ua = d4(0.0), ub = d4(0.0);
      if (va) {
        a0 = ldv(F.src + ga);
        if (F.vm2) a1 = ldv(F.vm2 + ga);
        if (F.vm1) a2 = ldv(F.vm1 + ga);
        if (ca < nE1)
          ua = Step::kStageHs ? make_double4(__ldg(S.hs + ga), 0.0, 0.0, 0.0)
                                : ldv_nc(S.lin + ga);
      }
      if (vb) {
        b0 = ldv(F.src + gb);
        if (F.vm2) b1 = ldv(F.vm2 + gb);
        if (F.vm1) b2 = ldv(F.vm1 + gb);
        if (cb < nE1)
          ub = Step::kStageHs ? make_double4(__ldg(S.hs + gb), 0.0, 0.0, 0.0)
                                : ldv_nc(S.lin + gb);
      }
      if (EIK_BAR1 && base == 0 && k > 0) __syncthreads();  // previous tile's step 3 done
      if (va) {
        const double4 x = form_x(F, a0, a1, a2);
        sst(ts.x, ca, x);
        if (ca < nE1) sst(ts.U, ca, ua);
        if (F.out && ca < nT) {
          if (EIK_L2POL) stv_pol(F.out + ga, x, pol_evict_last());
          else stv(F.out + ga, x);
        }
      }
      if (vb) {
        const double4 x = form_x(F, b0, b1, b2);
        sst(ts.x, cb, x);
        if (cb < nE1) sst(ts.U, cb, ub);
        if (F.out && cb < nT) {
          if (EIK_L2POL) stv_pol(F.out + gb, x, pol_evict_last());
          else stv(F.out + gb, x);
        }
      }
    }
    // row threadIdx.x of the tile: step 2's first row and, for an own cell, step 3's
    // (EIK_ROW0: loaded before the barrier that ends step 1 and kept)
    Row8 row0;
    Lrow lr0;
    const bool has0 = (int)threadIdx.x < nE1;
    if (EIK_ROW0 && has0) {
      row0 = load_row8(rows + (int64_t)threadIdx.x * 8);
      if (!Step::kE1Only) lr0 = load_lrow(lce1 + (int64_t)threadIdx.x * 6);
    }
    __syncthreads();
    SRP_MARK(0)
    if (EIK_PF4) {
      const int ln = (nT * 32 + 127) >> 7;
      const int nv = F.epi_vm1 ? 2 * ln : ln;
      // nv <= 2 * ceil(TPB * 32 / 128) <= TPB lines: one predicated prefetch per thread
      const int q = threadIdx.x;
      if (q < nv)
        prefetch_l1(q < ln ? (const char*)(S.ne + c0) + ((int64_t)q << 7)
                           : (const char*)(F.epi_vm1 + c0) + ((int64_t)(q - ln) << 7));
    }
    // step 2: L x on E1 (difference form; rows and coefficients contiguous
    // per tile), two rows per thread per round with their loads issued first
    auto lap_row = [&](int c, const Row8& row, const Lrow& lr) {
      const double4 xc = sld(ts.x, c);
      double4 acc = d4(0.0);
#pragma unroll
      for (int s = 0; s < KCMAX; ++s) {
        const double l = lr.v[s];
        const double4 xv = sld(ts.x, row.s[s]);
        acc.x += l * (xv.x - xc.x);
        acc.y += l * (xv.y - xc.y);
        acc.z += l * (xv.z - xc.z);
        acc.w += l * (xv.w - xc.w);
      }
      sst(ts.La, c, acc);
    };
    if (!Step::kE1Only) {
      if (EIK_PF5 && EIK_PF5A > 0 && (int)threadIdx.x < nT) {
        const double* cp = ctile + threadIdx.x;
#pragma unroll
        for (int q = 0; q < EIK_PF5A && q < NCOEF; ++q) prefetch_l2(cp + (int64_t)q * cstr);
      }
      if (EIK_ROW0) {
        if (has0) lap_row(threadIdx.x, row0, lr0);
        for (int c = threadIdx.x + TPB; c < nE1; c += TPB)
          lap_row(c, load_row8(rows + (int64_t)c * 8), load_lrow(lce1 + (int64_t)c * 6));
      } else {
        for (int c = threadIdx.x; c < nE1; c += TPB)
          lap_row(c, load_row8(rows + (int64_t)c * 8), load_lrow(lce1 + (int64_t)c * 6));
      }
      if (EIK_PF5 && (int)threadIdx.x < nT) {
        // step 3's first coefficient chunk into L2 while the CTA's last rows finish
        const double* cp = ctile + threadIdx.x;
#pragma unroll
        for (int q = EIK_PF5A; q < EIK_PF5A + EIK_PF5N && q < NCOEF; ++q)
          prefetch_l2(cp + (int64_t)q * cstr);
      }
      __syncthreads();
    }
    SRP_MARK(1)
    // step 3: z = scale * J x on the own cells
    if (EIK_PFT && k + 1 < kt) {
      nxt = load_meta(tile_of(k + 1));
      // the next tile's halo map (nE2 ints) into L2 while step 3 streams
      const int* nmap = S.e2map + nxt.e2off;
      const int nl = (nxt.nE2 * 4 + 127) >> 7;
      for (int q = threadIdx.x; q < nl; q += TPB) prefetch_l2((const char*)nmap + ((int64_t)q << 7));
    }
#if EIK_SMETA && EIK_PFM
    if (k + 1 < kt && (k + 1) % SMW != 0) {
      // the next tile's halo map into L1 while step 3 streams
      const TileMeta nm = smeta(k + 1);
      const int nl = ((Step::kE1Only ? nm.nE1 : nm.nE2) * 4 + 127) >> 7;
      if ((int)threadIdx.x < nl)
        prefetch_l1((const char*)(S.e2map + nm.e2off) + ((int64_t)threadIdx.x << 7));
    }
#endif
    if ((int)threadIdx.x < nT) {
      const int c = threadIdx.x;
      const int64_t i = c0 + c;
      const double4 ai = sld(ts.x, c);
      const double4 Ui = sld(ts.U, c);
      const double4 lai = Step::kE1Only ? d4(0.0) : sld(ts.La, c);
      const Row8 row = EIK_ROW0 ? row0 : load_row8(rows + (int64_t)c * 8);
      const Lrow lr = Step::kE1Only ? Lrow{}
                                    : (EIK_ROW0 ? lr0 : load_lrow(lce1 + (int64_t)c * 6));
      const double4 z = step(S, ts, row.s, lr.v, i, CoefPtr{ctile + c, cstr}, ai, Ui, lai);
      const double4 vm = F.epi_vm1 ? ldv(F.epi_vm1 + i) : d4(0.0);
      epi(i, z, ai, vm);
    }
    // the tile's shared arrays are rewritten by the next tile's step 1
    if (!EIK_BAR1) __syncthreads();
    SRP_MARK(2)
  }
  if (EIK_BAR1) __syncthreads();
#if EIK_PROF
  if (S.prof && threadIdx.x == 0) {
    for (int k = 0; k < 3; ++k) atomicAdd(S.prof + k, (unsigned long long)pst[k]);
    atomicAdd(S.prof + 3, 1ull);
  }
#endif
#undef SRP_MARK
}

template <class Epi>
__device__ __forceinline__ void swe_tiled(Smem& sm, const SweOp& S, const Form& F,
                                          const Epi& epi) {
  swe_tiled_op(sm, S, F, JvStep{}, epi);
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

// Host-callback operator (the reference's MatvecOperator around an arbitrary
// callable, phipm.py:45-54): the engine stays on the device and every matvec
// is a round trip to the host.  All CTAs write their part of x to the device
// buffer xd and arrive on a device counter; the lead thread posts a request
// sequence number in a mailbox in mapped pinned memory and spins (nanosleep)
// until the host thread serving eik_cb_phipm has copied x out (DMA on its own
// stream), called the callable, copied y = A x into yd and echoed the number
// (or an abort code); the engine's grid barrier after op_pre then releases
// every CTA to read yd (L2, bypassing L1).  Slow by construction (PCIe + the
// callable per matvec), as SURVEY.md §8(b)(1) allows for this plug point.
struct HostOp {
  static constexpr bool kTiled = false;
  int64_t n, NUu;
  double* xh;                     // device buffer x (n doubles), copied out by the host
  const double* yh;               // device buffer y = A x, copied in by the host
  volatile unsigned int* mbox;    // mapped: [0] request seq, [1] reply seq / kCbAbort
  unsigned long long* ctr;        // device: [0] CTA arrivals, [1] requests posted
  int* abort;                     // device: 1 once the host aborted (or timed out)
  unsigned long long timeout_ns;  // a request unanswered for this long aborts the call
  double scale;
  __device__ __forceinline__ int64_t NU() const { return NUu; }
};
constexpr unsigned int kCbAbort = 0xFFFFFFFFu;
constexpr unsigned long long kCbTimeoutNs = 600ull * 1000000000ull;  // default (EIK_CB_TIMEOUT_S)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

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

__device__ __forceinline__ void op_pre(const HostOp&, const double4*, double,
                                       int64_t, int64_t) {}

// op_pre with the exact vector the matvec is applied to (`formed`: v_j =
// raw / h already written by this thread for u in [lo, hi)); only the host
// operator needs it, the others recompute from raw and inv.
template <class Op>
__device__ __forceinline__ void op_pre_x(const Op& op, const double4* raw, double inv,
                                         const double4* formed, int64_t lo, int64_t hi) {
  op_pre(op, raw, inv, lo, hi);
}
template <>
__device__ __forceinline__ void op_pre_x<HostOp>(const HostOp& H, const double4*, double,
                                                 const double4* formed, int64_t lo,
                                                 int64_t hi) {
  if (*((volatile int*)H.abort)) return;
  for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
    const double4 a = formed[u];
    const double c[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * u + q < H.n) H.xh[4 * u + q] = c[q];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(H.ctr, 1ull);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long k = H.ctr[1] + 1;
    const unsigned long long target = k * gridDim.x;
    while (atomicAdd(H.ctr, 0ull) < target) __nanosleep(64);
    H.ctr[1] = k;
    __threadfence_system();
    const unsigned int seq = (unsigned int)(k & 0x7FFFFFFFu);
    H.mbox[0] = seq;
    __threadfence_system();
    const unsigned long long t0 = globaltimer_ns();
    unsigned int r;
    while ((r = H.mbox[1]) != seq && r != kCbAbort) {
      __nanosleep(2000);
      if (globaltimer_ns() - t0 > H.timeout_ns) { r = kCbAbort; break; }
    }
    if (r == kCbAbort) *((volatile int*)H.abort) = 1;
    __threadfence();
  }
}

__device__ __forceinline__ double4 op_main(const HostOp& H, const double4*, int64_t u) {
  double r[4] = {0.0, 0.0, 0.0, 0.0};
  if (!*((volatile int*)H.abort)) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * u + q < H.n) r[q] = H.scale * __ldcg(H.yh + 4 * u + q);
  }
  return make_double4(r[0], r[1], r[2], r[3]);
}

// true once a host-operator call was aborted (uniform after a grid barrier)
template <class Op>
__device__ __forceinline__ bool op_aborted(const Op&) { return false; }
template <>
__device__ __forceinline__ bool op_aborted<HostOp>(const HostOp& H) {
  return *((volatile int*)H.abort) != 0;
}

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
// Block-level degree-13 Pade with scaling and squaring (kernels.py:119-145)
// and LU with partial pivoting (LAPACK dgesv semantics: first max |pivot|,
// reciprocal scaling), run by one CTA of NT threads.  Matrices are n x n,
// row-major with a leading dimension ld = n rounded up to 4, plus 1,
// in shared memory when they fit (the dedicated dense kernel) or else in the
// L2-resident global scratch.  Every output of a product is one FMA chain
// over k in ascending order, whatever the layout.

__host__ __device__ constexpr int dense_ld(int n) { return ((n + 3) & ~3) + 1; }  // = 1 mod 4

struct DenseRed {
  double red[32];
  int ival;
  int piv[kDenseCap];     // blk_solve: pivot row of each elimination step
  double dg[kDenseCap];   // blk_solve: pivot values
  double rinv[kDenseCap]; // blk_solve: their reciprocals
};

// C = A B; C must not alias A or B.  Thread -> 4 x 4 output block
// (consecutive threads walk down the block rows, so with ld = 1 mod 4 the
// four A-column loads of a warp are conflict-free and the B-row loads are
// broadcasts); 16 FMA chains per thread, k ascending in each.
template <int NT>
__device__ void blk_matmul(const double* A, const double* B, double* C, int n, int ld) {
  const int nb = (n + 3) >> 2;
  for (int s = threadIdx.x; s < nb * nb; s += NT) {
    const int bj = s / nb, bi = s - bj * nb;
    const int i0 = 4 * bi, j0 = 4 * bj;
    const int ni = min(4, n - i0), nj = min(4, n - j0);
    const double* a = A + (int64_t)i0 * ld;
    const double* b = B + j0;
    double c[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) c[r][q] = 0.0;
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = r < ni ? a[(int64_t)r * ld + k] : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = q < nj ? b[(int64_t)k * ld + q] : 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[r][q] += av[r] * bv[q];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (r < ni && q < nj) C[(int64_t)(i0 + r) * ld + j0 + q] = c[r][q];
  }
  __syncthreads();
}

// max_j sum_i |M[i][j]|, rows summed in ascending order (numpy axis-0 reduce)
template <int NT>
__device__ double blk_norm1(DenseRed& rs, const double* M, int n, int ld) {
  double best = 0.0;
  for (int j = threadIdx.x; j < n; j += NT) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += fabs(M[(int64_t)i * ld + j]);
    best = fmax(best, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) rs.red[w] = best;
  __syncthreads();
  double r = 0.0;
  for (int q = 0; q < NT / 32; ++q) r = fmax(r, rs.red[q]);
  __syncthreads();
  return r;
}

// Solve P X = Q (Q <- X; P is destroyed): Gauss-Jordan elimination with
// partial pivoting (first index of max |P[r][k]| among the rows not yet
// pivoted, like LAPACK's idamax) done in place with implicit row
// interchanges, so an elimination step is one barrier: every warp finds the
// pivot redundantly, then eliminates column k from its own rows (pivot row
// read-only in that step).  Equivalent to dgesv's LU + substitution up to
// rounding.  The reference calls np.linalg.solve(V - U, V + U)
// (kernels.py:142).
template <int NT>
__device__ void blk_solve(DenseRed& rs, double* P, double* Q, int n, int ld) {
  static_assert(NT >= 64 && NT % 32 == 0, "blk_solve: at least two warps");
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned used = 0u;  // warp 0, bit q: row lane + 32 q is a pivot row already
  // pivot of column k (warp 0): |P[r][k]| compared as IEEE bit patterns
  // (monotonic for x >= 0), reduced with three 32-bit warp reductions
  auto pivot = [&](int k) {
    unsigned long long key = 0ull;
    int bi = n;
    for (int q = 0; lane + 32 * q < n; ++q) {
      const int r = lane + 32 * q;
      if ((used >> q) & 1u) continue;
      const unsigned long long b =
          (unsigned long long)__double_as_longlong(fabs(P[(int64_t)r * ld + k]));
      if (bi == n || b > key) { key = b; bi = r; }
    }
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned hmax = __reduce_max_sync(0xffffffffu, bi < n ? hi : 0u);
    const unsigned lmax = __reduce_max_sync(0xffffffffu, (bi < n && hi == hmax) ? lo : 0u);
    const bool cand = bi < n && hi == hmax && lo == lmax;
    const int pw = (int)__reduce_min_sync(0xffffffffu, cand ? (unsigned)bi : 0xffffffffu);
    if ((pw & 31) == lane) used |= 1u << (pw >> 5);
    if (lane == 0) {
      const double pk = P[(int64_t)pw * ld + k];
      rs.piv[k] = pw;
      rs.dg[k] = pk;
      rs.rinv[k] = 1.0 / pk;
    }
  };
  if (w == 0) pivot(0);
  __syncthreads();
  // step k (one barrier): warp 0 eliminates column k+1 first and finds the
  // next pivot from it (lookahead) while warps 1.. eliminate the other
  // columns (P k+2 .. n-1, then Q 0 .. n-1); lanes -> columns, warps -> rows.
  // Column k and the pivot row are only read in step k.
  for (int k = 0; k < n; ++k) {
    const int p = rs.piv[k];
    const double rinv = rs.rinv[k];
    if (w == 0) {
      if (k + 1 < n) {
        const double pv = P[(int64_t)p * ld + k + 1];
        for (int r = lane; r < n; r += 32)
          if (r != p) {
            double* x = P + (int64_t)r * ld;
            x[k + 1] = x[k + 1] - (x[k] * rinv) * pv;
          }
        __syncwarp();
        pivot(k + 1);
      }
    } else {
      const int np = n - k - 2;  // P columns k+2 .. n-1
      const int nc = (np > 0 ? np : 0) + n;
      for (int c0 = 0; c0 < nc; c0 += 4 * 32) {
        double* col[4];
        double pv[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + lane + 32 * q;
          ok[q] = c < nc;
          col[q] = c < np ? P + (k + 2 + c) : Q + (c - (np > 0 ? np : 0));
          pv[q] = ok[q] ? col[q][(int64_t)p * ld] : 0.0;
        }
        for (int r = w - 1; r < n; r += NW - 1) {
          if (r == p) continue;
          const double l = P[(int64_t)r * ld + k] * rinv;
          double v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = ok[q] ? col[q][(int64_t)r * ld] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (ok[q]) col[q][(int64_t)r * ld] = v[q] - l * pv[q];
        }
      }
    }
    __syncthreads();
  }
  // X[k] = Q[piv[k]] / pivot_k, staged through P's storage
  for (int idx = threadIdx.x; idx < n * n; idx += NT) {
    const int k = idx / n, j = idx - k * n;
    P[(int64_t)k * ld + j] = Q[(int64_t)rs.piv[k] * ld + j] / rs.dg[k];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += NT) {
    const int k = idx / n, j = idx - k * n;
    Q[(int64_t)k * ld + j] = P[(int64_t)k * ld + j];
  }
  __syncthreads();
}

// exp(M[0]) for the n x n matrix in M[0] (six matrices of n x ld scratch);
// returns the matrix holding the result.
template <int NT>
__device__ double* blk_expm(DenseRed& rs, double* const* M, int n, int ld) {
  const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0, 129060195264000.0, 10559470521600.0,
                        670442572800.0, 33522128640.0, 1323241920.0, 40840800.0,
                        960960.0, 16380.0, 182.0, 1.0};
  const int nn = n * ld;
  const double nrm = blk_norm1<NT>(rs, M[0], n, ld);
  int s = 0;
  if (nrm > kPadeTheta) {
    const double c = ceil(log2(nrm / kPadeTheta));
    s = c > 0.0 ? (int)c : 0;
  }
  const double sc = ldexp(1.0, s);
  if (s > 0) {
    for (int idx = threadIdx.x; idx < nn; idx += NT) M[0][idx] = M[0][idx] / sc;
    __syncthreads();
  }
  double *X = M[0], *X2 = M[1], *X4 = M[2], *X6 = M[3];
  blk_matmul<NT>(X, X, X2, n, ld);
  blk_matmul<NT>(X2, X2, X4, n, ld);
  blk_matmul<NT>(X2, X4, X6, n, ld);
  double* T = M[4];
  for (int idx = threadIdx.x; idx < nn; idx += NT)
    T[idx] = b[13] * X6[idx] + b[11] * X4[idx] + b[9] * X2[idx];
  __syncthreads();
  double* T2 = M[5];
  blk_matmul<NT>(X6, T, T2, n, ld);
  for (int idx = threadIdx.x; idx < nn; idx += NT) {
    const int i = idx / ld, j = idx - i * ld;
    T2[idx] = T2[idx] + b[7] * X6[idx] + b[5] * X4[idx] + b[3] * X2[idx] +
              (i == j ? b[1] : 0.0);
  }
  __syncthreads();
  double* U = M[4];  // T is dead
  blk_matmul<NT>(X, T2, U, n, ld);
  double* T3 = M[5];  // T2 is dead
  for (int idx = threadIdx.x; idx < nn; idx += NT)
    T3[idx] = b[12] * X6[idx] + b[10] * X4[idx] + b[8] * X2[idx];
  __syncthreads();
  double* V = M[0];  // X is dead
  blk_matmul<NT>(X6, T3, V, n, ld);
  for (int idx = threadIdx.x; idx < nn; idx += NT) {
    const int i = idx / ld, j = idx - i * ld;
    const double v = V[idx] + b[6] * X6[idx] + b[4] * X4[idx] + b[2] * X2[idx] +
                     (i == j ? b[0] : 0.0);
    const double u = U[idx];
    M[1][idx] = v - u;  // P (X2 dead after this loop: read before write per idx)
    M[2][idx] = v + u;  // Q (X4 likewise)
  }
  __syncthreads();
  blk_solve<NT>(rs, M[1], M[2], n, ld);
  int cur = 2, oth = 3;
  for (int q = 0; q < s; ++q) {
    blk_matmul<NT>(M[cur], M[cur], M[oth], n, ld);
    const int t = cur; cur = oth; oth = t;
  }
  return M[cur];
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
  int64_t dsm_bytes;        // dynamic shared memory per CTA (dense phase scratch)
};


// phi coefficients of one attempt (phipm.py:186-196, kernels.py:148-193):
// Hhat = [[H_keep, e_1, 0], [0, 0, I_{p-1}], [0, 0, 0]] of dimension
// keep + p + 1, E = exp(tau Hhat); writes phi[i] = E[i][keep+p-1] / tau^p
// (i < keep), phi[keep] = E[keep-1][keep+p] (the error corner) and
// phi[keep+1] = tau ||Hhat||_1.  `buf`: 6 * dim * dense_ld(dim) doubles.
template <int NT>
__device__ void dense_phi(DenseRed& rs, const EngineWork& Wk, double* buf, int64_t keep, int p,
                          double tau) {
  const int dim = (int)(keep + p + 1);
  const int ld = dense_ld(dim);
  const int64_t ldh = Wk.m_alloc;
  double* M[6];
  for (int q = 0; q < 6; ++q) M[q] = buf + (int64_t)q * dim * ld;
  double* M0 = M[0];
  for (int idx = threadIdx.x; idx < dim * ld; idx += NT) {
    const int i = idx / ld, jj = idx - i * ld;
    double hv = 0.0;
    if (i < keep && jj < keep) hv = Wk.H[i * ldh + jj];
    else if (i == 0 && jj == keep) hv = 1.0;
    else if (i >= keep && jj == i + 1 && i < keep + p) hv = 1.0;
    M0[idx] = hv;  // Hhat (zero padding columns)
  }
  __syncthreads();
  const double nrm_hat = blk_norm1<NT>(rs, M0, dim, ld);
  for (int idx = threadIdx.x; idx < dim * ld; idx += NT) M0[idx] = tau * M0[idx];
  __syncthreads();
  const double* Ex = blk_expm<NT>(rs, M, dim, ld);
  const double tp = pow(tau, (double)p);
  const int colp = p >= 1 ? (int)keep + p - 1 : 0;
  for (int i = threadIdx.x; i < keep; i += NT) Wk.phi[i] = Ex[(int64_t)i * ld + colp] / tp;
  if (threadIdx.x == 0) {
    Wk.phi[keep] = Ex[(int64_t)(keep - 1) * ld + keep + p];
    Wk.phi[keep + 1] = eik_mul(tau, nrm_hat);
  }
  __threadfence();
  __syncthreads();
}

// shared-memory budget of the dedicated dense kernel
constexpr int kDenseNT = 256;
constexpr size_t kDenseKernelSmem = 220 * 1024;
__host__ __device__ constexpr bool dense_fits_smem(int dim) {
  return (size_t)6 * dim * dense_ld(dim) * 8 <= kDenseKernelSmem;
}

// Result of an IOM2 sweep: kept dimension, breakdown flag, h_{m+1,m} and the
// recipe for v_{m+1} = ((vz - h1 vm1) - h2 vv) / hnext (or vz / hnext).
struct KrylovState {
  int64_t keep;
  bool broke;
  double hnext;
  const double4* vz;
  const double4* vm1;
  const double4* vv;
  double h1, h2;
  bool expl;
};

// IOM2 (krylov.py:53-112) with one tiled pass + one grid barrier per
// iteration: v_j is formed on the fly from (z_{j-1}, v_{j-2}, v_{j-1}) with
// the previous iteration's MGS coefficients; its norm comes from the Gram
// identity (explicit orthogonalisation pass only when that would cancel).
// H (row-major, leading dimension m_alloc) is written by CTA 0.
__device__ KrylovState krylov_tiled(cg::grid_group& grid, Smem& sm, const SweOp& op,
                                    const EngineWork& Wk, const double4* wp, double beta,
                                    int64_t m_eff, int64_t& mv_out) {
  int64_t mv = 0;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int64_t NU = Wk.NU, ld = Wk.m_alloc;
  int64_t lo, hi;
  brange(NU, lo, hi);
  KrylovState out;
  out.keep = m_eff;
  out.broke = false;
  out.hnext = 0.0;
  out.vz = Wk.zbuf;
  out.vm1 = nullptr;
  out.vv = nullptr;
  out.h1 = out.h2 = 0.0;
  out.expl = true;
  double hcur = beta;
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
          Form F;
          F.src = j == 0 ? wp : zin;
          F.vm2 = (j == 0 || expl) ? nullptr : vm2;
          F.vm1 = (j == 0 || expl) ? nullptr : vm1;
          F.a1 = a1;
          F.a2 = a2;
          F.h = hc;
          F.out = vj;
          F.epi_vm1 = vm1;
          F.rev = (int)(j & 1);
          swe_tiled(
              sm, op, F,
              [&](int64_t i, double4 z, double4 x, double4 b) {
                if (EIK_L2POL) stv_pol(zout + i, z, pol_evict_last());
                else stv(zout + i, z);
                d[1] += dot4(x, z);
                d[3] += dot4(z, z);
                d[4] += dot4(x, x);
                if (vm1) {
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
            out.broke = true;
            out.keep = j + 1;
            out.hnext = 0.0;
            break;
          }
          if (j + 1 < m_eff) {
            if (lead) Wk.H[(j + 1) * ld + j] = h;
            hcur = h;
            h1 = h1n;
            h2 = h2n;
          } else {
            out.hnext = h;
            out.vz = zout;
            out.h1 = h1n;
            out.h2 = h2n;
            out.vm1 = vm1;
            out.vv = vj;
            out.expl = expl;
          }
        }
  mv_out += mv;
  return out;
}

// ---------------------------------------------------------------- engine
// phipm_simul_iom2 (phipm.py:291-370) as a resumable state machine.  Every
// thread of every CTA runs the controller redundantly on identical values,
// so its state needs no broadcast: each thread keeps it in local memory
// (`EngineState`, accessed through a volatile reference so that none of it
// holds registers across the Krylov sweep).  The split step (k_swe_cont /
// k_swe_sweep in eik_api.cu) hands the state from kernel to kernel through
// global memory, written by the lead thread; the monolithic kernels run the
// sweep inline.
enum { EM_ATTEMPT = 0, EM_SWEEP, EM_AFTER_SWEEP };
enum { ER_DONE = 0, ER_SWEEP, ER_FAIL, ER_CONTINUE };

struct alignas(8) EngineState {
  // controller (phipm.py:318-359)
  double t, t_out, tau, tau_nom;
  int64_t m, m_cap, attempts, acc, rej, mv, nnz;
  const double4* y;
  int mode, p, io, y_nz, ycur, hits;
  unsigned vnzm;  // bit l: v_l is nonzero
  int wp_nz;
  // current attempt: Krylov input w_p / beta and the sweep's result
  const double4* wp;
  double beta;
  int64_t m_eff, keep;
  double hnext, h1, h2;
  const double4* vz;
  const double4* vm1;
  const double4* vv;
  int broke, expl;
};
using ES = volatile EngineState;
static_assert(sizeof(EngineState) % 8 == 0, "EngineState is copied as 8-byte words");

template <class T>
__device__ __forceinline__ void words_load(volatile T& dst, const T* src) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  volatile unsigned long long* d = reinterpret_cast<volatile unsigned long long*>(&dst);
  for (int k = 0; k < (int)(sizeof(T) / 8); ++k) d[k] = __ldcg(s + k);
}
template <class T>
__device__ __forceinline__ void words_store(T* dst, const volatile T& src) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  const volatile unsigned long long* s = reinterpret_cast<const volatile unsigned long long*>(&src);
  for (int k = 0; k < (int)(sizeof(T) / 8); ++k) __stcg(d + k, s[k]);
}

// Exact nonzero flags of v_l (the reference's vl.any()), warm-start seeds and
// the initial (tau, m) (phipm.py:300-317).  Returns false -- W = 0 written,
// info marked skipped -- when every v_l is zero (integrators.py:125-127).
__device__ bool eng_prologue(cg::grid_group& grid, Smem& sm, const EngineTask& T,
                             const EngineWork& Wk, int64_t nnz, ES& E) {
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int p = T.p;
  int64_t lo, hi;
  brange(Wk.NU, lo, hi);
  unsigned mask = 0;
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
#pragma unroll
    for (int l = 0; l < MAXV; ++l)
      if ((l <= p) && T.v[l] && c[l] > 0.0) mask |= 1u << l;
  }
  if (!mask) {
    for (int i = 0; i < T.ns; ++i)
      for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) T.W[i][u] = d4(0.0);
    if (lead) {
      EikPhipmInfo inf = {};
      inf.skipped = 1;
      Wk.info[T.info_idx] = inf;
    }
    grid.sync();
    return false;
  }
  double tau0 = T.tau_init;
  int64_t m0 = T.m_init;
  if (T.slot >= 0) {
    tau0 = __ldcg(Wk.seeds + 2 * T.slot);
    m0 = (int64_t)__ldcg(Wk.seeds + 2 * T.slot + 1);
  }
  double tau_i;
  int64_t m_i;
  const int64_t n = Wk.n;
  initial_tau_m(tau0, m0, T.rho[0], T.rho[T.ns - 1], T.m_max, n, &tau_i, &m_i);
  E.mode = EM_ATTEMPT;
  E.p = p;
  E.vnzm = mask;
  E.nnz = nnz;
  E.m_cap = T.m_max < n ? T.m_max : n;
  E.tau = tau_i;
  E.m = m_i;
  E.y = (mask & 1u) ? T.v[0] : Wk.zero;
  E.y_nz = (mask & 1u) ? 1 : 0;
  E.ycur = -1;
  E.t = 0.0;
  E.io = 0;
  E.t_out = T.rho[0];
  E.attempts = E.acc = E.rej = E.mv = 0;
  return true;
}

// A failed call: counters and status (EIK_EPHIPM: attempt budget exhausted,
// phipm.py:321-330; EIK_EINVAL: dense size cap) into the call's info record.
__device__ void eng_fail(cg::grid_group& grid, const EngineTask& T, const EngineWork& Wk, ES& E,
                         int status) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    EikPhipmInfo inf = {};
    inf.substeps = E.acc;
    inf.rejections = E.rej;
    inf.matvecs = E.mv;
    inf.tau_final = E.tau;
    inf.m_final = E.m;
    inf.t_reached = E.t;
    inf.attempts = E.attempts;
    inf.status = status;
    Wk.info[T.info_idx] = inf;
  }
  __threadfence();
  grid.sync();
}
__device__ __forceinline__ int eng_fail_status(const EngineTask& T, const EngineWork& Wk) {
  return __ldcg(&Wk.info[T.info_idx].status);
}

// Next attempt: write finished output points, then the w recurrence
// (phipm.py:159-182) and the Krylov set-up.  ER_DONE: every output written;
// ER_FAIL: attempt budget exhausted (info written); ER_SWEEP: the tiled IOM2
// sweep is due (the caller runs it inline or as its own kernel);
// ER_CONTINUE: the decomposition is complete here (generic operators, or a
// zero w_p), dense phase next.
template <class Op>
__device__ int eng_attempt(cg::grid_group& grid, Smem& sm, const Op& op, const EngineTask& T,
                           const EngineWork& Wk, ES& E) {
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int64_t NU = Wk.NU, n = Wk.n, ld = Wk.m_alloc;
  int64_t lo, hi;
  brange(NU, lo, hi);
  for (;;) {
    if (E.io >= T.ns) return ER_DONE;
    if (E.t < E.t_out) break;
    const double4* y = E.y;
    double4* Wo = T.W[E.io];
    for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) Wo[u] = y[u];
    E.io = E.io + 1;
    if (E.io < T.ns) E.t_out = T.rho[E.io];
  }
  if (op_aborted(op)) {
    eng_fail(grid, T, Wk, E, EIK_ECALLBACK);
    return ER_FAIL;
  }
  E.attempts = E.attempts + 1;
  if (E.attempts > T.max_attempts) {
    E.attempts = E.attempts - 1;
    eng_fail(grid, T, Wk, E, EIK_EPHIPM);
    return ER_FAIL;
  }
  E.tau_nom = E.tau;
  {
    const bool hits = eik_add(E.t, E.tau) >= E.t_out;
    E.hits = hits ? 1 : 0;
    if (hits) E.tau = eik_sub(E.t_out, E.t);
  }

  ProfClock pc;
  // ---- w recurrence (phipm.py:159-182)
  const int p = E.p;
  const unsigned vnzm = E.vnzm;
  const double t = E.t;
  const double4* wprev = E.y;
  bool wprev_nz = E.y_nz != 0;
  double ssq = 0.0;
  int64_t mv = 0;
  for (int j = 1; j <= p; ++j) {
    double cl[MAXV];
    for (int ell = 0; ell <= p - j; ++ell) cl[ell] = pow_over_fact(t, ell);
    const bool do_mv = !(T.zero_skip && !wprev_nz);
    double4* wj = Wk.w[j];
    double r[2] = {0.0, 0.0};
    bool tiled_mv = false;
    if constexpr (Op::kTiled) tiled_mv = op.tiled_ok && do_mv;
    if constexpr (Op::kTiled) {
      if (tiled_mv) {
        ++mv;
        // directions alternate back from the sweep's first iteration (rev 0):
        // every pass starts on the tiles the previous one streamed last
        Form F{wprev, nullptr, nullptr, 0.0, 0.0, 1.0, nullptr, nullptr, (p - j + 1) & 1};
        swe_tiled(sm, op, F,
                  [&](int64_t i, double4 z, double4, double4) {
                    double4 a = z;
                    for (int ell = 0; ell <= p - j; ++ell)
                      if ((vnzm >> (j + ell)) & 1u) a = a + cl[ell] * T.v[j + ell][i];
                    wj[i] = a;
                    r[0] += nz4(a);
                    r[1] += dot4(a, a);
                  });
      }
    }
    if (!tiled_mv) {
      if (do_mv) {
        op_pre_x(op, wprev, 1.0, wprev, lo, hi);
        grid.sync();
        ++mv;
      }
      for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) {
        double4 a = do_mv ? op_main(op, wprev, u) : d4(0.0);
        for (int ell = 0; ell <= p - j; ++ell)
          if ((vnzm >> (j + ell)) & 1u) a = a + cl[ell] * T.v[j + ell][u];
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
      const double4 a = wprev[u];
      r[0] += nz4(a);
      r[1] += dot4(a, a);
    }
    grid_reduce<2>(grid, sm, r, Wk.part);
    wprev_nz = r[0] > 0.0;
    ssq = r[1];
  }
  E.wp = wprev;
  E.wp_nz = wprev_nz ? 1 : 0;
  pc.mark(PC_WREC);

  // ---- IOM2 Krylov decomposition (krylov.py:53-112)
  E.beta = 0.0;
  E.hnext = 0.0;
  E.broke = 0;
  E.keep = 0;
  // v_{m+1} = ((vz - h1 vm1) - h2 vv) / hnext (tiled sweep) or vz / hnext
  E.vz = Wk.zbuf;
  E.vm1 = nullptr;
  E.vv = nullptr;
  E.h1 = E.h2 = 0.0;
  E.expl = 1;
  if (!wprev_nz) {
    E.mv = E.mv + mv;
    return ER_CONTINUE;
  }
  const double beta = sqrt(ssq);
  E.beta = beta;
  const int64_t m_eff = E.m < n ? E.m : n;
  const int64_t iom = m_eff < n ? T.iom : n;
  if (m_eff + p + 1 > MAXDIM || m_eff > Wk.m_alloc) {
    // kernels.py:159-163 raises ValueError once the augmented matrix would
    // exceed DENSE_SIZE_CAP (256); the basis holds at most 255 - p vectors
    E.mv = E.mv + mv;
    eng_fail(grid, T, Wk, E, EIK_EINVAL);
    return ER_FAIL;
  }
  E.m_eff = m_eff;
  E.keep = m_eff;
  if (blockIdx.x == 0) {
    for (int64_t q = threadIdx.x; q < m_eff * ld; q += TPB) Wk.H[q] = 0.0;
    __syncthreads();
  }
  if constexpr (Op::kTiled) {
    if (iom == 2 && op.tiled_ok) {
      E.mv = E.mv + mv;
      return ER_SWEEP;
    }
  }
  // generic operators: one matvec and one MGS pass per iteration
  double hcur = beta;
  const double4* raw = wprev;
  for (int64_t j = 0; j < m_eff; ++j) {
    double4* vj = Wk.basis + j * NU;
    const double4* vjm = j > 0 ? Wk.basis + (j - 1) * NU : nullptr;
    // v_j = raw / h (exact division), La = L v_j
    for (int64_t u = lo + threadIdx.x; u < hi; u += TPB) vj[u] = div4(raw[u], hcur);
    op_pre_x(op, raw, 1.0 / hcur, vj, lo, hi);
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
      E.broke = 1;
      E.keep = j + 1;
      E.hnext = 0.0;
      break;
    }
    if (j + 1 < m_eff) {
      // zbuf is complete: the reduction above ended with grid.sync
      if (lead) Wk.H[(j + 1) * ld + j] = h;
      hcur = h;
      raw = Wk.zbuf;
    } else {
      E.hnext = h;
    }
  }
  E.mv = E.mv + mv;
  pc.mark(PC_KRYLOV);
  return ER_CONTINUE;
}

__device__ __forceinline__ void eng_store_sweep(ES& E, const KrylovState& ks, int64_t kmv) {
  E.keep = ks.keep;
  E.broke = ks.broke ? 1 : 0;
  E.hnext = ks.hnext;
  E.vz = ks.vz;
  E.vm1 = ks.vm1;
  E.vv = ks.vv;
  E.h1 = ks.h1;
  E.h2 = ks.h2;
  E.expl = ks.expl ? 1 : 0;
  E.mv = E.mv + kmv;
  E.mode = EM_AFTER_SWEEP;
}

// Dense phi of the augmented Hessenberg matrix (kernels.py:148-193), the
// candidate (phipm.py:198-212, krylov.py:136-145) and the step-size / order
// controller (phipm.py:336-359).
// dense_ready: phi already in Wk.phi (the split step's k_swe_dense).
template <class Op>
__device__ void eng_finish_attempt(cg::grid_group& grid, Smem& sm, const Op& op,
                                   const EngineTask& T, const EngineWork& Wk, ES& E,
                                   bool dense_ready = false) {
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int64_t NU = Wk.NU, n = Wk.n;
  int64_t lo, hi;
  brange(NU, lo, hi);
  ProfClock pc;
  const int p = E.p;
  const double tau = E.tau;
  const bool wp_nz = E.wp_nz != 0;
  const bool broke = E.broke != 0;
  const int64_t keep = E.keep;
  const double beta = E.beta, hnext = E.hnext;
  double eps = 0.0, nh = 0.0, corner = 0.0;
  if (wp_nz) {
    if (!dense_ready) {
      __threadfence();
      grid.sync();
      if (blockIdx.x == 0) {
        // the tile buffers are dead here: the matrices go to dynamic shared
        // memory (past its 128-byte header) when they fit
        extern __shared__ __align__(128) unsigned char dsm[];
        __shared__ DenseRed rs;
        const int dim = (int)(keep + p + 1);
        const bool fits = (int64_t)6 * dim * dense_ld(dim) * 8 + 128 <= Wk.dsm_bytes;
        double* buf = fits ? reinterpret_cast<double*>(dsm + 128) : Wk.scr;
        dense_phi<TPB>(rs, Wk, buf, keep, p, tau);
      }
      grid.sync();
    }
    for (int i = threadIdx.x; i < keep + 2; i += TPB) sm.phi[i] = __ldcg(Wk.phi + i);
    __syncthreads();
    corner = sm.phi[keep];
    nh = sm.phi[keep + 1];
    pc.mark(PC_DENSE);
    eps = broke ? 0.0 : eik_mul(eik_mul(beta, fabs(hnext)), fabs(corner));
  }

  // the acceptance test needs only eps (phipm.py:336-341): the candidate is
  // formed for accepted attempts only (a rejected one never reads it)
  const bool accept = eik_div(eik_mul(E.t_out, eps), eik_mul(tau, T.tol)) <= T.delta;

  // ---- candidate (phipm.py:198-212, krylov.py:136-145)
  const int ycur = E.ycur;
  double4* cand = Wk.ybuf[ycur == 0 ? 1 : 0];
  bool cand_nz = false;
  if (accept) {
    const double4* y = E.y;
    const double4* vz = E.vz;
    const double4* vm1 = E.vm1;
    const double4* vv = E.vv;
    const double h1 = E.h1, h2 = E.h2;
    const bool expl = E.expl != 0;
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
#pragma unroll kCandU
        for (int64_t k = 0; k < keep; ++k) s = s + sm.phi[k] * Wk.basis[k * NU + u];
        double4 ap = beta * s;
        if (!broke) {
          double4 zz = vz[u];
          if (!expl) {
            if (vm1) zz = zz - h1 * vm1[u];
            zz = zz - h2 * vv[u];
          }
          ap = ap + corr * div4(zz, hnext);
        }
        c = c + tp * ap;
      }
      cand[u] = c;
      r[0] += nz4(c);
    }
    grid_reduce<1>(grid, sm, r, Wk.part);
    cand_nz = r[0] > 0.0;
  }
  pc.mark(PC_CAND);

  // ---- controller (phipm.py:336-359)
  const double t = E.t, t_out = E.t_out;
  const int64_t m = E.m, attempts = E.attempts;
  const double omega = eik_div(eik_mul(t_out, eps), eik_mul(tau, T.tol));
  const bool ok = omega <= T.delta;
  if (lead && Wk.trace) {
    // the trace is unbounded (phipm.py:341-343): trace_len counts every
    // attempt, rows beyond the buffer are dropped and the host re-runs the
    // (deterministic) call with a buffer of trace_len rows
    if (attempts <= Wk.trace_cap) {
      EikTraceRec tr;
      tr.attempt = attempts;
      tr.t = t;
      tr.tau = tau;
      tr.m = m;
      tr.eps_m = eps;
      tr.omega = omega;
      tr.accepted = ok ? 1 : 0;
      Wk.trace[attempts - 1] = tr;
    }
    *Wk.trace_len = attempts;
  }
  Adapt ad = adapt_parameters(tau, m, t, eps, nh, t_out, T.rho[T.ns - 1], p, T.tol, T.delta,
                              T.m_max, n, E.nnz);
  if (ok) {
    const bool hits = E.hits != 0;
    E.y = cand;
    E.ycur = ycur == 0 ? 1 : 0;
    E.y_nz = cand_nz ? 1 : 0;
    E.t = hits ? t_out : eik_add(t, tau);
    E.acc = E.acc + 1;
    if (hits && ad.tau < E.tau_nom) ad.tau = E.tau_nom;
  } else {
    E.rej = E.rej + 1;
  }
  E.tau = ad.tau > 1e-16 ? ad.tau : 1e-16;
  const int64_t m_cap = E.m_cap;
  E.m = ad.m < 1 ? 1 : (ad.m > m_cap ? m_cap : ad.m);
  E.mode = EM_ATTEMPT;
}

// Call summary and warm-start seeds (phipm.py:361-370).
__device__ void eng_epilogue(cg::grid_group& grid, const EngineTask& T, const EngineWork& Wk,
                             ES& E) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    EikPhipmInfo inf = {};
    inf.substeps = E.acc;
    inf.rejections = E.rej;
    inf.matvecs = E.mv;
    inf.tau_final = E.tau;
    inf.m_final = E.m;
    inf.t_reached = E.t;
    inf.attempts = E.attempts;
    inf.status = EIK_OK;
    Wk.info[T.info_idx] = inf;
    if (T.slot >= 0) {
      Wk.seeds[2 * T.slot] = E.tau;
      Wk.seeds[2 * T.slot + 1] = (double)E.m;
    }
  }
  __threadfence();
  grid.sync();
}

// One whole engine call in one kernel (the sweep inline); returns an
// eik_status, uniformly in every CTA.
template <class Op>
__device__ int engine_call(cg::grid_group& grid, Smem& sm, const Op& op,
                           const EngineTask& T, const EngineWork& Wk, int64_t nnz) {
  EngineState state;
  ES& E = state;
  if (!eng_prologue(grid, sm, T, Wk, nnz, E)) return EIK_OK;
  for (;;) {
    const int r = eng_attempt(grid, sm, op, T, Wk, E);
    if (r == ER_DONE) {
      eng_epilogue(grid, T, Wk, E);
      return EIK_OK;
    }
    if (r == ER_FAIL) return eng_fail_status(T, Wk);
    if constexpr (Op::kTiled) {
      if (r == ER_SWEEP) {
        ProfClock pc;
        int64_t kmv = 0;
        const KrylovState ks = krylov_tiled(grid, sm, op, Wk, E.wp, E.beta, E.m_eff, kmv);
        eng_store_sweep(E, ks, kmv);
        pc.mark(PC_KRYLOV);
      }
    }
    eng_finish_attempt(grid, sm, op, T, Wk, E);
  }
}

}  // namespace eik
