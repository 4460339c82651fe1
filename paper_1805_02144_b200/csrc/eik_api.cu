// eik_api.cu -- kernels and the C ABI (include/eik.h) of libeik.so.
//
// Host side owns: the ELL stencil built from the reference's CSR operators,
// device buffers, one CUDA stream per context, cooperative launches and the
// CUDA graph of a whole integrator step.  No compute runs on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "eik_dev.cuh"

using namespace eik;

// ====================================================================== errors
static thread_local std::string g_err;

// While a host-callback engine (eik_cb_phipm) is running, its cooperative
// kernel occupies every SM and waits for the host: a device-synchronising
// call made meanwhile (cudaFree in a destroy run by a finaliser or garbage
// collector inside the callable) would wait for that kernel and deadlock.
// Destroys are therefore deferred until the engine call has finished, and
// libeik entry points called from inside the callable fail with EIK_EINVAL.
static std::atomic<int> g_cb_inflight{0};
static thread_local bool g_in_callback = false;
static std::mutex g_defer_mu;
static std::vector<std::function<void()>> g_deferred;
#define EIK_NO_REENTRY()                                                                   \
  if (g_in_callback)                                                                       \
  return fail(EIK_EINVAL, "libeik called from inside a matvec callback (the device engine " \
                          "is waiting for it)")
static bool defer_destroy(std::function<void()> fn) {
  std::lock_guard<std::mutex> lk(g_defer_mu);
  if (g_cb_inflight.load() == 0) return false;
  g_deferred.push_back(std::move(fn));
  return true;
}
static void drain_deferred() {
  std::vector<std::function<void()>> todo;
  {
    std::lock_guard<std::mutex> lk(g_defer_mu);
    if (g_cb_inflight.load() != 0) return;
    todo.swap(g_deferred);
  }
  for (auto& f : todo) f();
}
#ifndef EIK_LPT
#define EIK_LPT 0
#endif
// dynamic smem floor: the dense phase keeps its 6 matrices in shared memory
// for n = m + p + 1 <= 46
static constexpr size_t kDenseSmemBytes = 128 + (size_t)6 * 46 * dense_ld(46) * 8;
static eik_status fail(eik_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(EIK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ====================================================================== kernels

__device__ __forceinline__ void smem_init(Smem& sm) {
  if (threadIdx.x == 0) {
    sm.par = 0;
  }
  __syncthreads();
}

// (u_x; u_y; u_z; h) SoA  <->  per-cell double4
// (user cell order, see the device cell order in eik_swe_create: device cell
// i is user cell ord[i])
__global__ void k_soa_to_cell(const double* __restrict__ s, double4* d, int64_t N,
                              const int* __restrict__ ord) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = ord[i];
    d[i] = make_double4(s[u], s[N + u], s[2 * N + u], s[3 * N + u]);
  }
}
__global__ void k_cell_to_soa(const double4* __restrict__ d, double* s, int64_t N,
                              const int* __restrict__ ord) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double4 v = d[i];
    const int64_t u = ord[i];
    s[u] = v.x;
    s[N + u] = v.y;
    s[2 * N + u] = v.z;
    s[3 * N + u] = v.w;
  }
}

// Saved position of a split step between kernels (written by the lead thread
// of the kernel that hands over, read by every thread of the next one).
struct alignas(8) StepState {
  EngineState E;
  EngineTask T;
  int64_t nA;
  const double4* base;
  const double4* fin;
  int call;
  int more;  // host-loop mode: the loop condition (the graph uses `cond`)
};

struct SweArgs {
  SweOp S1;   // J at the linearisation state (scale 1)
  SweOp SD;   // dt * J (the engine operator, integrators.py:117)
  EngineWork Wk;
  // step buffers
  double4 *u, *uprev, *fn, *v1, *va, *vb, *d2, *Ub, *W[5];
  // API buffers
  double4 *x, *out;
  double dt, tol;
  double c09cube;      // 0.9 ** 3 as CPython computes it
  int scheme;
  int* status;         // device status word
  double* nnz_out;
  double* dbg;         // optional per-row output (nnz per cell)
  EngineTask task;     // engine-level API
  // split step graph
  StepState* ss;                    // saved step position (global)
  cudaGraphConditionalHandle cond;  // loop condition of the graph's while node
  int resume;                       // 0: first k_swe_cont of the step
  int hostloop;                     // 1: no graph; the host reads ss->more
};

// F(w) (+ eta at w when `lin` is w); optional out_v = dt * F.
// returns a status uniform over the grid.
__device__ int phase_rhs(cg::grid_group& grid, Smem& sm, const SweOp& S,
                         const double4* w, double4* out_f, double4* out_v,
                         double dt, bool write_eta, double* part) {
  int64_t lo, hi;
  brange(S.N, lo, hi);
  SrcPtr src{w};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) S.lapA[i] = swe_lap_cell(S, src, i);
  grid.sync();
  double r[1] = {0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) {
    double eta;
    const double4 F = swe_rhs_cell(S, src, S.lapA, i, &eta);
    if (write_eta) {
      const double4 q = S.nf[i];
      S.ne[i] = make_double4(q.x, q.y, q.z, eta);
    }
    if (out_f) out_f[i] = F;
    if (out_v) out_v[i] = dt * F;
    r[0] += nf4(F) + nf4(w[i]);
  }
  grid_reduce<1>(grid, sm, r, part);
  return r[0] > 0.0 ? EIK_ENONFINITE : EIK_OK;
}

// F(u_n), eta and v_1 = dt F(u_n) at the start of a step: one tiled pass on
// the compact stencil when it is valid (the API-level F keeps the CSR-order
// phase_rhs, which reproduces scipy's csr_matvec order)
__device__ int phase_rhs_step(cg::grid_group& grid, Smem& sm, const SweOp& S, const double4* u,
                              double4* out_f, double4* out_v, double dt, double* part) {
  if (!S.tiled_ok) return phase_rhs(grid, sm, S, u, out_f, out_v, dt, true, part);
  double r[1] = {0.0};
  Form FA{u, nullptr, nullptr, 0.0, 0.0, 1.0, nullptr, nullptr};
  swe_tiled_op(sm, S, FA, RhsStep{true, true}, [&](int64_t i, double4 F, double4 w, double4) {
    out_f[i] = F;
    out_v[i] = dt * F;
    r[0] += nf4(F) + nf4(w);
  });
  grid_reduce<1>(grid, sm, r, part);
  return r[0] > 0.0 ? EIK_ENONFINITE : EIK_OK;
}

// d = (F(U) - f_n) - J (U - u_n)   (integrators.py:101-102), epilogue(i, d)
template <class Epi>
__device__ int phase_dev(cg::grid_group& grid, Smem& sm, const SweOp& S,
                         const double4* U, const double4* fn, Epi epi,
                         double* part, const double4* Uadd = nullptr,
                         double4* Ubuf = nullptr, bool keep_U = false) {
  if (S.tiled_ok) {
    // one 1-ring tiled pass: [F*(U) - J*_n U] - g_n (DevStep); with Uadd the
    // stage state U + Uadd is formed on the fly, (U - (-1) Uadd) / 1 being
    // exactly U + Uadd
    double r[1] = {0.0};
    // (keep_U: U + Uadd is also stored to Ubuf, every cell being own in one tile)
    Form FD{U, Uadd, nullptr, -1.0, 0.0, 1.0, (Uadd && keep_U) ? Ubuf : nullptr, nullptr};
    swe_tiled_op(sm, S, FD, DevStep{}, [&](int64_t i, double4 d, double4 w, double4) {
      epi(i, d);
      r[0] += nf4(d) + nf4(w);
    });
    grid_reduce<1>(grid, sm, r, part);
    return r[0] > 0.0 ? EIK_ENONFINITE : EIK_OK;
  }
  if (Uadd) {
    pointwise(S.N, [&](int64_t i) { Ubuf[i] = U[i] + Uadd[i]; });
    grid.sync();
    U = Ubuf;
  }
  int64_t lo, hi;
  brange(S.N, lo, hi);
  SrcPtr su{U};
  SrcDiff sx{U, S.lin};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) {
    S.lapA[i] = swe_lap_cell(S, su, i);
    S.lapB[i] = swe_lap_cell(S, sx, i);
  }
  grid.sync();
  double r[1] = {0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) {
    double eta;
    const double4 F = swe_rhs_cell(S, su, S.lapA, i, &eta);
    const double4 Jx = swe_jv_cell(S, sx, S.lapB, i);
    const double4 d = (F - fn[i]) - Jx;
    epi(i, d);
    r[0] += nf4(F) + nf4(U[i]);
  }
  grid_reduce<1>(grid, sm, r, part);
  return r[0] > 0.0 ? EIK_ENONFINITE : EIK_OK;
}

// n_A = nnz of the assembled J = (J_v + J_r) + J_m with scipy's zero-dropping
// (swe.py:175-223).  Products and sums use _rn
// intrinsics so exact zeros come out exactly as in numpy.
__device__ double phase_count_nnz(cg::grid_group& grid, Smem& sm, const SweOp& S,
                                  double* part, double* per_row = nullptr) {
  int64_t lo, hi;
  brange(S.N, lo, hi);
  double r[1] = {0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) {
    const double4 Ui = S.lin[i];
    const int cn = __ldg(S.cnt + i);
    // eta exactly as numpy: ((Vx@ux + Vy@uy) + Vz@uz) + f, each csr_matvec
    // a sequential sum in column order, no FMA
    double sv[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < cn; ++s) {
      const double4 Uj = S.lin[S.nb(s, i)];
      sv[0] = __dadd_rn(sv[0], __dmul_rn(S.c(s, OP_VX, i), Uj.x));
      sv[1] = __dadd_rn(sv[1], __dmul_rn(S.c(s, OP_VY, i), Uj.y));
      sv[2] = __dadd_rn(sv[2], __dmul_rn(S.c(s, OP_VZ, i), Uj.z));
    }
    const double4 nfi = S.nf[i];
    const double4 q = make_double4(nfi.x, nfi.y, nfi.z,
                                   __dadd_rn(__dadd_rn(__dadd_rn(sv[0], sv[1]), sv[2]), nfi.w));
    const double P[3] = {__dsub_rn(__dmul_rn(q.y, Ui.z), __dmul_rn(q.z, Ui.y)),
                         __dsub_rn(__dmul_rn(q.z, Ui.x), __dmul_rn(q.x, Ui.z)),
                         __dsub_rn(__dmul_rn(q.x, Ui.y), __dmul_rn(q.y, Ui.x))};
    const double ex = __dmul_rn(q.w, q.x), ey = __dmul_rn(q.w, q.y),
                 ez = __dmul_rn(q.w, q.z);
    // Jr off-diagonal blocks (a,b): xy +ez, xz -ey, yx -ez, yz +ex, zx +ey, zy -ex
    const double rot[3][3] = {{0.0, ez, -ey}, {-ez, 0.0, ex}, {ey, -ex, 0.0}};
    double c = 4.0 * (double)__ldg(S.dfx + i);
    for (int s = 0; s < cn; ++s) {
      const int64_t j = S.nb(s, i);
      const double4 Uj = S.lin[j];
      const double uj[3] = {Uj.x, Uj.y, Uj.z};
      const double df = __ldg(S.df1 + (int64_t)s * S.N + i);
      double G[3], D[3], V[3];
      for (int k = 0; k < 3; ++k) {
        G[k] = S.c(s, OP_GX + k, i);
        D[k] = S.c(s, OP_DX + k, i);
        V[k] = S.c(s, OP_VX + k, i);
      }
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) {
          const double jv = -__dmul_rn(P[a], V[b]);
          const double jr = (a == b) ? df : (j == i ? rot[a][b] : 0.0);
          const double jm = -__dmul_rn(G[a], uj[b]);
          c += (__dadd_rn(__dadd_rn(jv, jr), jm) != 0.0);
        }
        c += (G[a] != 0.0);  // -(g G_a) block
      }
      for (int b = 0; b < 3; ++b) c += (__dmul_rn(D[b], Uj.w) != 0.0);
      const double t = __dadd_rn(__dadd_rn(__dmul_rn(D[0], uj[0]), __dmul_rn(D[1], uj[1])),
                                 __dmul_rn(D[2], uj[2]));
      c += (__dadd_rn(__dadd_rn(0.0, df), -t) != 0.0);
    }
    if (per_row) per_row[i] = c;
    r[0] += c;
  }
  grid_reduce<1>(grid, sm, r, part);
  return r[0];
}

__device__ void set_status(int* st, int v) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *st = v;
}

template <class F>
__device__ void pointwise(int64_t N, F f) {
  int64_t lo, hi;
  brange(N, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) f(i);
}

// PhiTask's default m_max (phipm.py:87-107), used by every step-path call
constexpr int64_t kStepMMax = 100;

__device__ EngineTask base_task(const SweArgs& A) {
  EngineTask T;
  for (int l = 0; l < MAXV; ++l) T.v[l] = nullptr;
  for (int l = 0; l < MAXNS; ++l) T.W[l] = nullptr;
  T.tol = A.tol;
  T.delta = 1.4;
  T.tau_init = -1.0;
  T.m_init = 1;
  T.iom = 2;
  T.m_max = kStepMMax;
  T.max_attempts = 1000000;
  T.zero_skip = 1;
  return T;
}

// ---------------------------------------------------------------- step kernels
// One integrator step (integrators.py:140-224) on the resident state
// (A.S1: J at u_n, A.SD: dt*J, the engine operator).  Per engine call of the
// scheme: the stage work before it and its task; u_{n+1} = base + fin.
__device__ __forceinline__ int step_ncalls(int scheme) {
  return scheme == EIK_EXPRB53 ? 3 : (scheme >= EIK_EXPRB42 ? 2 : 1);
}

__device__ int step_call_setup(cg::grid_group& grid, Smem& sm, const SweArgs& A, int call,
                               EngineTask& T, const double4*& base, const double4*& fin) {
  const double dt = A.dt;
  const int scheme = A.scheme;
  const double4* u = A.u;
  double4* Ub = A.Ub;
  double4 *va = A.va, *vb = A.vb, *d2 = A.d2;
  double4* const* W = A.W;
  int st = EIK_OK;
  T = base_task(A);
  T.info_idx = call;
  T.ns = 1;
  T.rho[0] = 1.0;
  const int key = scheme * 4 + call;
  if (key == EIK_EPI3 * 4) {
    const double c = (2.0 / 3.0) * dt;
    st = phase_dev(grid, sm, A.S1, A.uprev, A.fn,
                   [&](int64_t i, double4 d) { va[i] = c * d; }, A.Wk.part);
  } else if (key == EIK_EXPRB42 * 4 + 1) {
    const double c = (32.0 / 9.0) * dt;
    st = phase_dev(grid, sm, A.S1, u, A.fn, [&](int64_t i, double4 d) { va[i] = c * d; },
                   A.Wk.part, W[0], Ub);
  } else if (key == EIK_PEXPRB43 * 4 + 1) {
    st = phase_dev(grid, sm, A.S1, u, A.fn, [&](int64_t i, double4 d) { d2[i] = d; },
                   A.Wk.part, W[0], Ub);
    if (st == EIK_OK) {
      st = phase_dev(grid, sm, A.S1, u, A.fn,  // U3 = u + W1
                     [&](int64_t i, double4 d3) {
                       const double4 a = d2[i];
                       va[i] = dt * ((16.0 * a) - (2.0 * d3));
                       vb[i] = dt * ((-48.0 * a) + (12.0 * d3));
                     },
                     A.Wk.part, W[1], Ub, true);  // Ub = U3: the base of u_{n+1}
    }
  } else if (key == EIK_EXPRB53 * 4 + 1) {
    st = phase_dev(grid, sm, A.S1, u, A.fn,
                   [&](int64_t i, double4 d) { d2[i] = d; va[i] = dt * d; }, A.Wk.part, W[0],
                   Ub);
  } else if (key == EIK_EXPRB53 * 4 + 2) {
    const double c1 = 27.0 / 25.0, c2 = 729.0 / 125.0, q3 = A.c09cube;
    pointwise(A.S1.N, [&](int64_t i) {
      const double4 w2 = W[2][i], w3 = W[3][i];
      const double4 ph = make_double4(w2.x / 0.125, w2.y / 0.125, w2.z / 0.125, w2.w / 0.125);
      const double4 pn = make_double4(w3.x / q3, w3.y / q3, w3.z / q3, w3.w / q3);
      Ub[i] = ((u[i] + W[1][i]) + c1 * ph) + c2 * pn;
    });
    grid.sync();
    const double e1 = 250.0 / 81.0, e2 = 500.0 / 27.0;
    st = phase_dev(grid, sm, A.S1, Ub, A.fn,
                   [&](int64_t i, double4 d3) {
                     const double4 a = d2[i];
                     va[i] = dt * ((18.0 * a) - (e1 * d3));
                     vb[i] = dt * ((-60.0 * a) + (e2 * d3));
                   },
                   A.Wk.part);
  }
  if (st != EIK_OK) return st;
  switch (key) {
    case EIK_RB_EULER * 4:
      T.p = 1; T.v[1] = A.v1; T.W[0] = W[0]; T.slot = EIK_SLOT_RBE;
      fin = W[0];
      break;
    case EIK_EPI3 * 4:
      T.p = 2; T.v[1] = A.v1; T.v[2] = va; T.W[0] = W[0]; T.slot = EIK_SLOT_EPI3;
      fin = W[0];
      break;
    case EIK_EXPRB42 * 4:
      T.p = 1; T.v[1] = A.v1; T.rho[0] = 0.75; T.W[0] = W[0]; T.slot = EIK_SLOT_EXPRB42_1;
      break;
    case EIK_EXPRB42 * 4 + 1:
      T.p = 3; T.v[1] = A.v1; T.v[3] = va; T.W[0] = W[1]; T.slot = EIK_SLOT_EXPRB42_2;
      fin = W[1];
      break;
    case EIK_PEXPRB43 * 4:
      T.p = 1; T.v[1] = A.v1; T.ns = 2; T.rho[0] = 0.5; T.rho[1] = 1.0;
      T.W[0] = W[0]; T.W[1] = W[1]; T.slot = EIK_SLOT_PEXPRB43_1;
      break;
    case EIK_PEXPRB43 * 4 + 1:
      T.p = 4; T.v[3] = va; T.v[4] = vb; T.W[0] = W[2]; T.slot = EIK_SLOT_PEXPRB43_2;
      fin = W[2];
      base = Ub;  // u_{n+1} = U3 + W2
      break;
    case EIK_EXPRB53 * 4:
      T.p = 1; T.v[1] = A.v1; T.ns = 2; T.rho[0] = 0.5; T.rho[1] = 0.9;
      T.W[0] = W[0]; T.W[1] = W[1]; T.slot = EIK_SLOT_EXPRB53_1;
      break;
    case EIK_EXPRB53 * 4 + 1:
      T.p = 3; T.v[3] = va; T.ns = 2; T.rho[0] = 0.5; T.rho[1] = 0.9;
      T.W[0] = W[2]; T.W[1] = W[3]; T.slot = EIK_SLOT_EXPRB53_2;
      break;
    case EIK_EXPRB53 * 4 + 2:
      T.p = 4; T.v[1] = A.v1; T.v[3] = va; T.v[4] = vb; T.W[0] = W[4];
      T.slot = EIK_SLOT_EXPRB53_3;
      fin = W[4];
      break;
    default:
      return EIK_EINVAL;
  }
  return EIK_OK;
}

// u_prev <- u_n, u_{n+1} = base + fin
__device__ void step_finish(const SweArgs& A, const double4* base, const double4* fin) {
  double4* uu = A.u;
  double4* up = A.uprev;
  pointwise(A.S1.N, [&](int64_t i) {
    const double4 old = uu[i];
    const double4 nb = base[i] + fin[i];
    up[i] = old;
    uu[i] = nb;
  });
}

// Monolithic step: one cooperative launch with every Krylov sweep inline
// (used when the split graph below is unavailable, or with EIK_STEP_MONO=1).
__global__ void __launch_bounds__(TPB, MINB) k_swe_step(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  ProfClock pc;
  int st = phase_rhs_step(grid, sm, A.S1, A.u, A.fn, A.v1, A.dt, A.Wk.part);
  pc.mark(PC_RHS);
  if (st != EIK_OK) { set_status(A.status, st); return; }
  // loop state in local memory: none of it may hold registers across sweeps
  volatile int64_t nA = (int64_t)phase_count_nnz(grid, sm, A.S1, A.Wk.part);
  pc.mark(PC_NNZ);
  const double4* volatile base = A.u;
  const double4* volatile fin = nullptr;
  __shared__ EngineTask sT;
  for (volatile int call = 0; call < step_ncalls(A.scheme) && st == EIK_OK; ++call) {
    EngineTask T;
    const double4* b = base;
    const double4* f = fin;
    st = step_call_setup(grid, sm, A, call, T, b, f);
    base = b;
    fin = f;
    pc.mark(PC_DEV);
    if (st != EIK_OK) break;
    // the task lives in shared memory during the call: its fields are read a
    // few times per attempt and must not occupy registers across the sweep
    if (threadIdx.x == 0) sT = T;
    __syncthreads();
    st = engine_call(grid, sm, A.SD, sT, A.Wk, nA);
    pc.skip();
  }
  if (st == EIK_OK) step_finish(A, base, fin);
  set_status(A.status, st);
}

// Split step (the default): the graph  cont ; while (cond) { sweep ; cont }.
// k_swe_cont runs the step from its saved position up to the next tiled
// Krylov sweep, saves the position and sets the loop condition; k_swe_sweep
// runs that sweep as a kernel of its own, so the sweep is compiled with the
// whole register budget and no controller state live across it.
__device__ void cont_stop(const SweArgs& A, int st) {
  set_status(A.status, st);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (A.hostloop) A.ss->more = 0;
    else cudaGraphSetConditional(A.cond, 0u);
  }
}

__global__ void __launch_bounds__(TPB, MINB) k_swe_cont(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  if (lead) atomicAdd(A.Wk.kiters + 2, 1ull);
  ProfClock pc;
  EngineState state;
  ES& E = state;
  __shared__ EngineTask sT;
  volatile int64_t nA;
  const double4* volatile base;
  const double4* volatile fin;
  volatile int call;
  volatile int in_engine;
  StepState* G = A.ss;
  if (!A.resume) {
    const int st = phase_rhs_step(grid, sm, A.S1, A.u, A.fn, A.v1, A.dt, A.Wk.part);
    pc.mark(PC_RHS);
    if (st != EIK_OK) { cont_stop(A, st); return; }
    nA = (int64_t)phase_count_nnz(grid, sm, A.S1, A.Wk.part);
    pc.mark(PC_NNZ);
    base = A.u;
    fin = nullptr;
    call = 0;
    in_engine = 0;
  } else {
    words_load(E, &G->E);
    if (threadIdx.x == 0) sT = G->T;
    nA = G->nA;
    base = G->base;
    fin = G->fin;
    call = G->call;
    in_engine = 1;
    __syncthreads();
    pc.skip();
    if (E.mode == EM_AFTER_SWEEP) eng_finish_attempt(grid, sm, A.SD, sT, A.Wk, E, true);
  }
  for (;;) {
    if (!in_engine) {
      if (call >= step_ncalls(A.scheme)) {
        step_finish(A, base, fin);
        cont_stop(A, EIK_OK);
        return;
      }
      EngineTask T;
      const double4* b = base;
      const double4* f = fin;
      const int st = step_call_setup(grid, sm, A, call, T, b, f);
      base = b;
      fin = f;
      pc.mark(PC_DEV);
      if (st != EIK_OK) { cont_stop(A, st); return; }
      if (threadIdx.x == 0) sT = T;
      __syncthreads();
      if (!eng_prologue(grid, sm, sT, A.Wk, nA, E)) {
        call = call + 1;
        continue;
      }
      in_engine = 1;
    }
    const int r = eng_attempt(grid, sm, A.SD, sT, A.Wk, E);
    if (r == ER_SWEEP) {
      // every CTA read G at entry and has passed a grid barrier since
      E.mode = EM_SWEEP;
      if (lead) {
        words_store(&G->E, E);
        G->T = sT;
        G->nA = nA;
        G->base = base;
        G->fin = fin;
        G->call = call;
        if (A.hostloop) G->more = 1;
        else cudaGraphSetConditional(A.cond, 1u);
      }
      return;
    }
    if (r == ER_FAIL) { cont_stop(A, eng_fail_status(sT, A.Wk)); return; }
    if (r == ER_DONE) {
      eng_epilogue(grid, sT, A.Wk, E);
      call = call + 1;
      in_engine = 0;
      continue;
    }
    eng_finish_attempt(grid, sm, A.SD, sT, A.Wk, E);
  }
}

// The dense phase of an attempt after a sweep: one CTA of kDenseNT threads
// with the matrices in shared memory (global scratch beyond ~68 x 68).
__global__ void __launch_bounds__(kDenseNT, 1) k_swe_dense(SweArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ DenseRed rs;
  if (threadIdx.x == 0) atomicAdd(A.Wk.kiters + 2, 1ull);
  ProfClock pc;
  const EngineState& E = A.ss->E;
  if (E.mode != EM_AFTER_SWEEP || !E.wp_nz) return;
  const int64_t keep = E.keep;
  const int p = E.p;
  const int dim = (int)(keep + p + 1);
  double* buf = dense_fits_smem(dim) ? reinterpret_cast<double*>(dsm) : A.Wk.scr;
  dense_phi<kDenseNT>(rs, A.Wk, buf, keep, p, E.tau);
  pc.mark(PC_DENSE);
}

__global__ void __launch_bounds__(TPB, MINB) k_swe_sweep(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  if (lead) atomicAdd(A.Wk.kiters + 2, 1ull);
  ProfClock pc;
  StepState* G = A.ss;
  const double4* wp = G->E.wp;
  const double beta = G->E.beta;
  const int64_t m_eff = G->E.m_eff;
  int64_t kmv = 0;
  const KrylovState ks = krylov_tiled(grid, sm, A.SD, A.Wk, wp, beta, m_eff, kmv);
  // every CTA read G before the sweep's first grid barrier
  if (lead) {
    ES& GE = G->E;
    eng_store_sweep(GE, ks, kmv);
  }
  pc.mark(PC_KRYLOV);
}

// ------------------------------------------------------- API-level kernels
__global__ void __launch_bounds__(TPB, MINB) k_swe_rhs(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  int st = phase_rhs(grid, sm, A.S1, A.x, A.out, nullptr, 0.0, false, A.Wk.part);
  set_status(A.status, st);
}

__global__ void __launch_bounds__(TPB, MINB) k_swe_jv(SweArgs A) {
  // A.x = linearisation state, A.va = direction, A.out = J v
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const SweOp& S = A.S1;
  int st = phase_rhs(grid, sm, S, A.x, A.fn, nullptr, 0.0, true, A.Wk.part);
  int64_t lo, hi;
  brange(S.N, lo, hi);
  op_pre(S, A.va, 1.0, lo, hi);
  grid.sync();
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) A.out[i] = op_main(S, A.va, i);
  set_status(A.status, st);
}

__global__ void __launch_bounds__(TPB, MINB) k_swe_nnz(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  int st = phase_rhs(grid, sm, A.S1, A.x, A.fn, nullptr, 0.0, true, A.Wk.part);
  const double c = phase_count_nnz(grid, sm, A.S1, A.Wk.part, A.dbg);
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.nnz_out = c;
  set_status(A.status, st);
}

__global__ void __launch_bounds__(TPB, MINB) k_swe_phipm(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  int st = phase_rhs(grid, sm, A.S1, A.x, A.fn, nullptr, 0.0, true, A.Wk.part);
  if (st != EIK_OK) { set_status(A.status, st); return; }
  const int64_t nA = (int64_t)phase_count_nnz(grid, sm, A.S1, A.Wk.part);
  st = engine_call(grid, sm, A.SD, A.task, A.Wk, nA);
  set_status(A.status, st);
}


// Krylov-loop microbenchmark: `reps` IOM2 sweeps of dimension A.scheme on the
// direction A.va at the linearisation state A.x (no controller, no expm).
__global__ void __launch_bounds__(TPB, MINB) k_swe_kbench(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const SweOp& S = A.SD;
  phase_rhs(grid, sm, A.S1, A.x, A.fn, nullptr, 0.0, true, A.Wk.part);
  int64_t lo, hi;
  brange(S.N, lo, hi);
  int64_t mv = 0;
  for (int r = 0; r < (int)A.tol; ++r) {
    double q[1] = {0.0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) q[0] += dot4(A.va[i], A.va[i]);
    grid_reduce<1>(grid, sm, q, A.Wk.part);
    if (S.tiled_ok) {
      KrylovState ks = krylov_tiled(grid, sm, S, A.Wk, A.va, sqrt(q[0]), A.scheme, mv);
      if (blockIdx.x == 0 && threadIdx.x == 0) *A.nnz_out = (double)ks.keep;
    }
  }
  set_status(A.status, EIK_OK);
}


// Conservation diagnostics (swe.py:226-237): weighted totals of mass h,
// energy g h + |u|^2/2 and potential enstrophy (zeta + f)^2 / (2 h), with
// zeta = V.u (no f: swe.py:233 subtracts it again).  Weights are per-cell
// areas (A.dbg) or, when null, the scalar A.tol (reference: ops.cell_area).
// Out: A.nnz_out[0..3] = mass, energy, enstrophy, count of h <= 0.
__global__ void __launch_bounds__(TPB, MINB) k_swe_diag(SweArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const SweOp& S = A.S1;
  const double4* u = A.x;
  int64_t lo, hi;
  brange(S.N, lo, hi);
  double r[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += TPB) {
    double zeta = 0.0;
    for (int s = 0; s < S.K; ++s) {
      const double4 uj = u[S.nb(s, i)];
      zeta += S.c(s, OP_VX, i) * uj.x + S.c(s, OP_VY, i) * uj.y + S.c(s, OP_VZ, i) * uj.z;
    }
    const double4 ui = u[i];
    const double f = S.nf[i].w;
    const double w = A.dbg ? A.dbg[i] : A.tol;
    const double eta = zeta + f;
    r[0] += w * ui.w;
    r[1] += w * (S.g * ui.w + 0.5 * (ui.x * ui.x + ui.y * ui.y + ui.z * ui.z));
    r[2] += w * (eta * eta / (2.0 * ui.w));
    r[3] += (ui.w <= 0.0) ? 1.0 : 0.0;
  }
  grid_reduce<4>(grid, sm, r, A.Wk.part);
  if (blockIdx.x == 0 && threadIdx.x < 4) A.nnz_out[threadIdx.x] = r[threadIdx.x];
  set_status(A.status, EIK_OK);
}

struct CsrArgs {
  CsrOp C;
  EngineWork Wk;
  EngineTask task;
  int* status;
};

__global__ void __launch_bounds__(TPB, MINB) k_csr_phipm(CsrArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const int st = engine_call(grid, sm, A.C, A.task, A.Wk, A.Wk.nnz);
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.status = st;
}

struct CbArgs {
  HostOp H;
  EngineWork Wk;
  EngineTask task;
  int* status;
};

__global__ void __launch_bounds__(TPB, MINB) k_cb_phipm(CbArgs A) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  const int st = engine_call(grid, sm, A.H, A.task, A.Wk, A.Wk.nnz);
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.status = st;
}

// ====================================================================== host

namespace {

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, count * sizeof(T) + 64);
}

struct Bufs {
  std::vector<void*> ptrs;
  template <class T>
  cudaError_t get(T** p, size_t count) {
    cudaError_t e = dalloc(p, count);
    if (e == cudaSuccess) {
      ptrs.push_back(*p);
      e = cudaMemset(*p, 0, count * sizeof(T));
    }
    return e;
  }
  // free *p (allocated here) and allocate count elements in its place
  template <class T>
  cudaError_t regrow(T** p, size_t count) {
    for (auto it = ptrs.begin(); it != ptrs.end(); ++it)
      if (*it == (void*)*p) {
        cudaFree(*it);
        ptrs.erase(it);
        break;
      }
    *p = nullptr;
    return get(p, count);
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
};

int coop_grid(const void* const* kernels, int nk, int dev, int64_t NU, size_t smem) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int best = 1 << 30;
  for (int k = 0; k < nk; ++k) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernels[k], TPB, smem);
    best = std::min(best, nb * nsm);
  }
  if (best < 1) return 0;
  const int64_t need = (NU + TPB - 1) / TPB;
  return (int)std::max<int64_t>(1, std::min<int64_t>(best, need));
}

// Recursive coordinate bisection of ord[lo, hi) into nt leaves of sizes
// differing by at most one; leaf starts are appended to `starts` in order.
// Each leaf is left sorted by user index (the grid's own locality order).
void rcb_order(const double* px, const double* py, const double* pz, int32_t* ord, int64_t lo,
               int64_t hi, int nt, std::vector<int32_t>& starts) {
  const int64_t n = hi - lo;
  if (nt <= 1 || n <= 1) {
    std::sort(ord + lo, ord + hi);
    starts.push_back((int32_t)lo);
    for (int k = 1; k < nt; ++k) starts.push_back((int32_t)hi);  // empty leaves
    return;
  }
  const int n1 = nt / 2;
  const int64_t k = (n * n1 + nt / 2) / nt;
  const double* P[3] = {px, py, pz};
  int ax = -1;
  double best = 0.0;
  for (int a = 0; a < 3; ++a) {
    double mn = P[a][ord[lo]], mx = mn;
    for (int64_t q = lo; q < hi; ++q) {
      mn = std::min(mn, P[a][ord[q]]);
      mx = std::max(mx, P[a][ord[q]]);
    }
    if (mx - mn > best) { best = mx - mn; ax = a; }
  }
  if (ax >= 0) {
    const double* c = P[ax];
    std::nth_element(ord + lo, ord + lo + k, ord + hi, [c](int32_t a, int32_t b) {
      return c[a] < c[b] || (c[a] == c[b] && a < b);
    });
  } else {
    std::sort(ord + lo, ord + hi);
  }
  rcb_order(px, py, pz, ord, lo, lo + k, n1, starts);
  rcb_order(px, py, pz, ord, lo + k, hi, nt - n1, starts);
}

}  // namespace

struct EngineHost {
  Bufs mem;
  int dev = 0;
  cudaStream_t st = nullptr;
  int G = 1;
  int64_t NU = 0, n = 0, m_alloc = 0;
  EngineWork wk{};
  double4* vin[MAXV] = {};
  double4* wout[MAXNS] = {};
  EikPhipmInfo* info_d = nullptr;
  EikTraceRec* trace_d = nullptr;
  int64_t trace_cap_d = 0;
  int64_t* trace_len_d = nullptr;
  int* status_d = nullptr;
  double* nnz_d = nullptr;
  unsigned long long* kiters_d = nullptr;
  int64_t launches = 0;

  size_t smem = 0;
  eik_status init(int device, int64_t NU_, int64_t n_, int64_t m_alloc_,
                  const void* const* kernels, int nk, size_t smem_bytes = 0,
                  int G_override = 0) {
    dev = device;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    NU = NU_;
    n = n_;
    m_alloc = std::max<int64_t>(1, m_alloc_);
    smem = smem_bytes;
    // the attribute is per function and process-wide: only ever raise it,
    // so contexts with smaller tiles never break a larger one's launches
    static std::map<const void*, size_t> attr_max;  // per kernel set
    size_t& cur = attr_max[kernels[0]];
    if (smem > cur) {
      for (int k = 0; k < nk; ++k)
        CK(cudaFuncSetAttribute(kernels[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
      cur = smem;
    }
    const int cap = coop_grid(kernels, nk, dev, 1LL << 40, smem);  // co-resident capacity
    G = coop_grid(kernels, nk, dev, NU, smem);
    wk.dsm_bytes = (int64_t)smem;
    if (G_override > 0) {
      if (G_override > cap)
        return fail(EIK_ECUDA, "cooperative grid does not fit the device");
      G = G_override;
    }
    CK(mem.get(&wk.basis, (size_t)m_alloc * NU));
    CK(mem.get(&wk.zbuf, NU));
    CK(mem.get(&wk.zbuf2, NU));
    for (int l = 1; l < MAXV; ++l) CK(mem.get(&wk.w[l], NU));
    CK(mem.get(&wk.ybuf[0], NU));
    CK(mem.get(&wk.ybuf[1], NU));
    CK(mem.get(&wk.zero, NU));
    CK(mem.get(&wk.part, (size_t)2 * NPART * part_stride(G)));
    CK(mem.get(&wk.H, (size_t)m_alloc * m_alloc));
    CK(mem.get(&wk.scr, (size_t)6 * MAXDIM * dense_ld(MAXDIM)));
    CK(mem.get(&wk.phi, MAXDIM + 4));
    CK(mem.get(&wk.seeds, 2 * EIK_NUM_SLOTS));
    CK(mem.get(&info_d, 4));
    CK(mem.get(&trace_len_d, 1));
    CK(mem.get(&status_d, 1));
    CK(mem.get(&nnz_d, 4));
    CK(mem.get(&kiters_d, 4));
    wk.info = info_d;
    wk.trace = nullptr;
    wk.trace_cap = 0;
    wk.trace_len = trace_len_d;
    wk.kiters = kiters_d;
    wk.NU = NU;
    wk.n = n;
    wk.m_alloc = m_alloc;
    return reset_seeds();
  }
  // grow the Krylov basis and H to m vectors (m <= min(n, MAXDIM))
  eik_status reserve(int64_t m) {
    m = std::min<int64_t>(std::min<int64_t>(m, n), MAXDIM);
    if (m <= m_alloc) return EIK_OK;
    CK(cudaSetDevice(dev));
    CK(cudaStreamSynchronize(st));
    CK(mem.regrow(&wk.basis, (size_t)m * NU));
    CK(mem.regrow(&wk.H, (size_t)m * m));
    m_alloc = m;
    wk.m_alloc = m;
    return EIK_OK;
  }
  eik_status reset_seeds() {
    std::vector<double> s(2 * EIK_NUM_SLOTS);
    for (int k = 0; k < EIK_NUM_SLOTS; ++k) {
      s[2 * k] = -1.0;  // None
      s[2 * k + 1] = 1.0;
    }
    CK(cudaMemcpy(wk.seeds, s.data(), s.size() * sizeof(double), cudaMemcpyHostToDevice));
    return EIK_OK;
  }
  eik_status ensure_io() {
    if (vin[0]) return EIK_OK;
    for (int l = 0; l < MAXV; ++l) CK(mem.get(&vin[l], NU));
    for (int l = 0; l < MAXNS; ++l) CK(mem.get(&wout[l], NU));
    return EIK_OK;
  }
  eik_status ensure_trace(int64_t cap) {
    if (cap <= trace_cap_d) return EIK_OK;
    if (trace_d) cudaFree(trace_d);
    CK(dalloc(&trace_d, (size_t)cap));
    trace_cap_d = cap;
    return EIK_OK;
  }
  // validation mirroring PhiTask.__post_init__ (phipm.py:109-125)
  eik_status check_task(const EikPhiTask* t) {
    if (!t) return fail(EIK_EINVAL, "task is NULL");
    if (t->p < 0 || t->p + 1 > MAXV)
      return fail(EIK_EINVAL, "at least one input vector is required (p+1 <= 8)");
    if (t->ns < 1 || t->ns > MAXNS || !t->rho)
      return fail(EIK_EINVAL, "rho must lie in (0, 1]");
    if (!(t->rho[0] > 0.0) || t->rho[t->ns - 1] > 1.0)
      return fail(EIK_EINVAL, "rho must lie in (0, 1]");
    for (int i = 1; i < t->ns; ++i)
      if (!(t->rho[i] > t->rho[i - 1])) return fail(EIK_EINVAL, "rho must be strictly ascending");
    if (!(t->tol > 0.0)) return fail(EIK_EINVAL, "tol must be positive");
    if (t->iom < 1) return fail(EIK_EINVAL, "iom must be >= 1");
    // m_cap = min(m_max, n) (phipm.py:302); the dense cap (kernels.py:20,
    // 159-163) is checked when the basis would outgrow it, as the reference
    // raises then, so the basis never needs more than MAXDIM vectors
    const int64_t mcap = std::min<int64_t>(std::min<int64_t>(std::max(t->m_max, 1), n), MAXDIM);
    if (mcap > m_alloc)
      return fail(EIK_EINVAL, "m_max exceeds the context's basis allocation");
    return EIK_OK;
  }
  EngineTask make_task(const EikPhiTask* t) {
    EngineTask T;
    memset(&T, 0, sizeof(T));
    T.p = t->p;
    T.ns = t->ns;
    for (int i = 0; i < t->ns; ++i) T.rho[i] = t->rho[i];
    for (int l = 0; l <= t->p; ++l) T.v[l] = (t->v && t->v[l]) ? vin[l] : nullptr;
    for (int i = 0; i < t->ns; ++i) T.W[i] = wout[i];
    T.tol = t->tol;
    T.delta = t->delta;
    T.tau_init = t->tau_init > 0.0 ? t->tau_init : -1.0;
    T.m_init = t->m_init;
    T.iom = t->iom;
    T.m_max = t->m_max;
    T.max_attempts = t->max_attempts > 0 ? t->max_attempts : 1000000;
    T.zero_skip = t->zero_skip;
    T.slot = -1;
    T.info_idx = 0;
    return T;
  }
  eik_status finish_phipm(EikPhipmInfo* info, EikTraceRec* trace, int64_t trace_cap,
                          int64_t* trace_len) {
    int sth = 0;
    EikPhipmInfo inf;
    CK(cudaMemcpyAsync(&sth, status_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&inf, info_d, sizeof(inf), cudaMemcpyDeviceToHost, st));
    int64_t tl = 0;
    CK(cudaMemcpyAsync(&tl, trace_len_d, sizeof(tl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (info) *info = inf;
    if (trace && trace_cap > 0) {
      const int64_t nrec = std::min(tl, trace_cap);
      if (nrec > 0)
        CK(cudaMemcpy(trace, trace_d, nrec * sizeof(EikTraceRec), cudaMemcpyDeviceToHost));
      if (trace_len) *trace_len = tl;
    } else if (trace_len) {
      *trace_len = 0;
    }
    if (sth == EIK_EPHIPM) return fail(EIK_EPHIPM, "no convergence within the substep budget");
    if (sth == EIK_EINVAL)
      return fail(EIK_EINVAL, "augmented dense size exceeds cap 256");
    if (sth != EIK_OK) return fail((eik_status)sth, "engine failed");
    return EIK_OK;
  }
  void release() {
    if (trace_d) cudaFree(trace_d);
    trace_d = nullptr;
    mem.release();
    if (st) cudaStreamDestroy(st);
    st = nullptr;
  }
};

struct EikSwe {
  EngineHost eng;
  int64_t N = 0;
  int K = 0;
  SweOp S{};
  double4 *u = nullptr, *uprev = nullptr, *fn = nullptr, *v1 = nullptr, *va = nullptr,
          *vb = nullptr, *d2 = nullptr, *Ub = nullptr, *W[5] = {}, *x = nullptr,
          *out = nullptr;
  double* soa = nullptr;
  double* wts = nullptr;  // diagnostics weights (lazily allocated)
  int* ord_d = nullptr;   // device cell -> user cell
  std::vector<int32_t> ord_h;
  bool have_prev = false;
  double c09cube = 0.0;
  // graph cache for eik_swe_step
  cudaGraphExec_t gexec = nullptr;
  int g_scheme = -1;
  double g_dt = 0.0, g_tol = 0.0;
  bool graphs_ok = true;
  bool split = getenv("EIK_STEP_MONO") == nullptr;  // split step graph
  StepState* ss = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // host-loop mode (no graph): the split step's kernels launched one by one,
  // the loop condition read back after every k_swe_cont; every Krylov sweep
  // is bracketed by CUDA events (sweep-kernel timing, ncu profiling)
  bool hostloop = getenv("EIK_STEP_HOST") != nullptr;
  cudaEvent_t evs0 = nullptr, evs1 = nullptr;
  double sweep_ms = 0.0;
  int64_t nsweeps = 0;
  bool sweep_log = getenv("EIK_SWEEP_LOG") != nullptr;
  unsigned long long kit_last = 0;
  float last_ms = 0.0f;
  double* pinned = nullptr;  // pinned staging for host copies (4N doubles)
  // eik_swe_snapshot: device copy of (u, u_prev, seeds)
  double4 *snap_u = nullptr, *snap_prev = nullptr;
  double* snap_seeds = nullptr;
  bool snap_have_prev = false;

  SweArgs args(double4* lin = nullptr, double dt = 1.0) {
    SweArgs A;
    memset(&A, 0, sizeof(A));
    A.S1 = S;
    A.S1.lin = lin ? lin : u;
    A.S1.scale = 1.0;
    A.SD = A.S1;
    A.SD.scale = dt;
    A.Wk = eng.wk;
    A.u = u;
    A.uprev = uprev;
    A.fn = fn;
    A.v1 = v1;
    A.va = va;
    A.vb = vb;
    A.d2 = d2;
    A.Ub = Ub;
    for (int k = 0; k < 5; ++k) A.W[k] = W[k];
    A.x = x;
    A.out = out;
    A.c09cube = c09cube;
    A.status = eng.status_d;
    A.nnz_out = eng.nnz_d;
    return A;
  }
  eik_status launch(const void* fn_, SweArgs& A) {
    void* kargs[] = {&A};
    CK(cudaLaunchCooperativeKernel(fn_, eng.G, TPB, kargs, eng.smem, eng.st));
    ++eng.launches;
    return EIK_OK;
  }
  eik_status h2d_cells(const double* h, double4* d) {
    CK(cudaMemcpyAsync(soa, h, 4 * N * sizeof(double), cudaMemcpyHostToDevice, eng.st));
    k_soa_to_cell<<<std::min<int64_t>((N + 255) / 256, 4096), 256, 0, eng.st>>>(soa, d, N, ord_d);
    ++eng.launches;
    CK(cudaGetLastError());
    return EIK_OK;
  }
  eik_status d2h_cells(const double4* d, double* h) {
    k_cell_to_soa<<<std::min<int64_t>((N + 255) / 256, 4096), 256, 0, eng.st>>>(d, soa, N, ord_d);
    ++eng.launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, soa, 4 * N * sizeof(double), cudaMemcpyDeviceToHost, eng.st));
    CK(cudaStreamSynchronize(eng.st));
    return EIK_OK;
  }
  eik_status status() {
    int sth = 0;
    CK(cudaMemcpyAsync(&sth, eng.status_d, sizeof(int), cudaMemcpyDeviceToHost, eng.st));
    CK(cudaStreamSynchronize(eng.st));
    if (sth == EIK_ENONFINITE) return fail(EIK_ENONFINITE, "non-finite right-hand side");
    if (sth == EIK_EPHIPM) return fail(EIK_EPHIPM, "no convergence within the substep budget");
    if (sth != EIK_OK) return fail((eik_status)sth, "device step failed");
    return EIK_OK;
  }
};

struct EikCsr {
  EngineHost eng;
  CsrOp C{};
  int64_t nnz = 0;
};

static const void* kSweKernels[] = {(const void*)k_swe_step, (const void*)k_swe_cont,
                                    (const void*)k_swe_sweep, (const void*)k_swe_rhs,
                                    (const void*)k_swe_jv, (const void*)k_swe_nnz,
                                    (const void*)k_swe_phipm, (const void*)k_swe_kbench,
                                    (const void*)k_swe_diag};
static const void* kCsrKernels[] = {(const void*)k_csr_phipm};
static const void* kCbKernels[] = {(const void*)k_cb_phipm};

struct EikCb {
  EngineHost eng;
  HostOp H{};
  double* xh = nullptr;  // pinned host staging of x and y
  double* yh = nullptr;
  unsigned int* mbox = nullptr;  // mapped pinned mailbox
  cudaStream_t cst = nullptr;    // copies while the engine kernel runs
};

extern "C" {

const char* eik_last_error(void) { return g_err.c_str(); }
int eik_version(void) { return 1; }

eik_status eik_tile_order(int64_t n, const double* px, const double* py, const double* pz,
                          int32_t ntiles, int32_t* ord, int32_t* starts) {
  if (n < 1 || n > INT32_MAX || ntiles < 1 || !px || !py || !pz || !ord || !starts)
    return fail(EIK_EINVAL, "invalid arguments to eik_tile_order");
  std::vector<int32_t> st;
  for (int64_t i = 0; i < n; ++i) ord[i] = (int32_t)i;
  rcb_order(px, py, pz, ord, 0, n, ntiles, st);
  st.push_back((int32_t)n);
  for (size_t t = 0; t < st.size(); ++t) starts[t] = st[t];
  return EIK_OK;
}

eik_status eik_swe_create(int32_t n_g, const EikCsrView* ops, const double* n_x,
                          const double* n_y, const double* n_z, const double* f,
                          const double* h_s, double g, double nu, int32_t device,
                          int32_t m_max, EikSwe** out) {
  EIK_NO_REENTRY();
  if (!out || !ops || n_g < 1 || !n_x || !n_y || !n_z || !f || !h_s)
    return fail(EIK_EINVAL, "invalid arguments to eik_swe_create");
  const int64_t N = n_g;
  // ---- union stencil per row, ELL coefficients.  Slots follow the sorted
  // column order of the CSR rows (self included at its sorted position) so
  // that sequential slot sums reproduce scipy's csr_matvec order exactly.
  std::vector<std::vector<int32_t>> cols(N);
  for (int64_t i = 0; i < N; ++i) cols[i].push_back((int32_t)i);
  for (int o = 0; o < NOPS; ++o) {
    const EikCsrView& M = ops[o];
    if (!M.indptr || (M.nnz > 0 && (!M.indices || !M.data)))
      return fail(EIK_EINVAL, "operator CSR arrays missing");
    if (M.indptr[N] != M.nnz) return fail(EIK_EINVAL, "operator indptr/nnz mismatch");
    for (int64_t i = 0; i < N; ++i)
      for (int32_t k = M.indptr[i]; k < M.indptr[i + 1]; ++k) {
        const int32_t j = M.indices[k];
        if (j < 0 || j >= N) return fail(EIK_EINVAL, "column index out of range");
        if (!std::isfinite(M.data[k])) return fail(EIK_EINVAL, "SparseMatrix entries must be finite");
        auto& c = cols[i];
        if (std::find(c.begin(), c.end(), j) == c.end()) c.push_back(j);
      }
  }
  int K = 1;
  for (int64_t i = 0; i < N; ++i) {
    std::sort(cols[i].begin(), cols[i].end());
    K = std::max<int>(K, (int)cols[i].size());
  }
  if (K > KMAX) return fail(EIK_EINVAL, "stencil wider than 8 points per row");
  std::vector<int32_t> nbr((size_t)K * N), cnt(N), dfx(N, 0);
  std::vector<double> coef((size_t)K * NOPS * N, 0.0), df1((size_t)K * N, 0.0);
  for (int64_t i = 0; i < N; ++i) {
    cnt[i] = (int32_t)cols[i].size();
    for (int s = 0; s < K; ++s)
      nbr[(size_t)s * N + i] = s < cnt[i] ? cols[i][s] : (int32_t)i;
  }
  auto slot_of = [&](int64_t i, int32_t j) -> int {
    const auto& c = cols[i];
    auto it = std::lower_bound(c.begin(), c.end(), j);
    if (it != c.end() && *it == j) return (int)(it - c.begin());
    return -1;
  };
  for (int o = 0; o < NOPS; ++o) {
    const EikCsrView& M = ops[o];
    for (int64_t i = 0; i < N; ++i)
      for (int32_t k = M.indptr[i]; k < M.indptr[i + 1]; ++k) {
        const int s = slot_of(i, M.indices[k]);
        coef[((size_t)s * NOPS + o) * N + i] += M.data[k];
      }
  }
  {
    const EikCsrView& Df = ops[10];
    if (!Df.indptr || Df.indptr[N] != Df.nnz)
      return fail(EIK_EINVAL, "Df CSR arrays missing or inconsistent");
    for (int64_t i = 0; i < N; ++i)
      for (int32_t k = Df.indptr[i]; k < Df.indptr[i + 1]; ++k) {
        const int s = slot_of(i, Df.indices[k]);
        if (s >= 0) df1[(size_t)s * N + i] += Df.data[k];
        else if (Df.data[k] != 0.0) dfx[i] += 1;
      }
  }
  // ---- Df contract.  The device applies Df u as -nu * L(L u) (no 2-ring
  // stencil streamed per Krylov iteration); the reference applies the given
  // Df matrix (swe.py:163-167, 190).  Accept only operator sets whose Df is
  // -nu * (L @ L): per entry |Df_ij + nu (LL)_ij| <= 1e-12 nu sum_k |L_ik L_kj|
  // (rounding of the product, whatever its summation order), entries outside
  // the pattern of L@L exactly zero.
  {
    const EikCsrView& L = ops[OP_L];
    const EikCsrView& Df = ops[10];
    std::vector<double> ll(N, 0.0), mag(N, 0.0), dv(N, 0.0);
    std::vector<char> seen(N, 0);
    std::vector<int32_t> touched;
    const double anu = std::fabs(nu);
    for (int64_t i = 0; i < N; ++i) {
      touched.clear();
      for (int32_t k = L.indptr[i]; k < L.indptr[i + 1]; ++k) {
        const int32_t j = L.indices[k];
        const double a = L.data[k];
        for (int32_t k2 = L.indptr[j]; k2 < L.indptr[j + 1]; ++k2) {
          const int32_t c2 = L.indices[k2];
          const double v = a * L.data[k2];
          ll[c2] += v;
          mag[c2] += std::fabs(v);
          if (!seen[c2]) { seen[c2] = 1; touched.push_back(c2); }
        }
      }
      for (int32_t k = Df.indptr[i]; k < Df.indptr[i + 1]; ++k) {
        const int32_t c2 = Df.indices[k];
        dv[c2] += Df.data[k];
        if (!seen[c2]) { seen[c2] = 1; touched.push_back(c2); }
      }
      bool ok = true;
      for (int32_t c2 : touched) {
        if (std::fabs(dv[c2] + nu * ll[c2]) > 1e-12 * anu * mag[c2]) ok = false;
        ll[c2] = mag[c2] = dv[c2] = 0.0;
        seen[c2] = 0;
      }
      if (!ok)
        return fail(EIK_EINVAL, "Df must equal -nu * (L @ L): the device applies it as "
                                "-nu * L(L u) (row " + std::to_string(i) + ")");
    }
  }
  // ---- device cell order.  The Krylov pass works on tiles of <= TILE own
  // cells plus their 2-ring halo; the cells are renumbered so that every tile
  // is a contiguous range of device cells forming a compact patch: recursive
  // coordinate bisection of the cell positions (n_x, n_y, n_z) into NT equal
  // leaves (median splits along the longest extent, ties by user index).
  // Degenerate positions (planar operators: n constant) keep the user order.
  // Slots keep the user rows' sorted column order, so every stencil sum runs
  // in scipy's order; only reductions over cells change their order.
  int nsm = 0;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return fail(EIK_ECUDA, "no CUDA device");
  const int Gt = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * MINB, (N + TILE - 1) / TILE));
  // the tile buffers of MINB co-resident CTAs must fit one SM's shared
  // memory: more, smaller tiles until they do
  int smem_sm = 0, smem_optin = 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const size_t smem_budget =
      std::min<size_t>((size_t)smem_optin, (size_t)smem_sm / MINB - 1024 - 4096);
  std::vector<int32_t> ord(N), tstart;
  int NT = 0;
  {
    std::vector<int32_t> mark(N, -1);
    // tiles per CTA: the fewest that keep every tile within TILE cells and the
    // shared-memory budget; EIK_TILES_EXTRA (environment, experiments) adds to it
    int64_t per0 = (N + (int64_t)Gt * TILE - 1) / ((int64_t)Gt * TILE);
    if (const char* e = getenv("EIK_TILES_EXTRA")) per0 += std::max(0, atoi(e));
    for (int64_t per = per0;; ++per) {
      NT = (int)(Gt * per);
      for (int64_t i = 0; i < N; ++i) ord[i] = (int32_t)i;
      tstart.clear();
      rcb_order(n_x, n_y, n_z, ord.data(), 0, N, NT, tstart);
      tstart.push_back((int32_t)N);
      int e1m = 1, e2m = 1;
      std::vector<int32_t> e1;
      for (int t = 0; t < NT; ++t) {
        e1.clear();
        int n1 = 0, n2 = 0;
        for (int32_t d = tstart[t]; d < tstart[t + 1]; ++d) mark[ord[d]] = t, ++n1;
        for (int32_t d = tstart[t]; d < tstart[t + 1]; ++d)
          for (int32_t j : cols[ord[d]])
            if (mark[j] != t) { mark[j] = t; e1.push_back(j); }
        n1 += (int)e1.size();
        n2 = n1;
        for (int32_t j1 : e1)
          for (int32_t j : cols[j1])
            if (mark[j] != t) { mark[j] = t; ++n2; }
        e1m = std::max(e1m, n1);
        e2m = std::max(e2m, n2);
      }
      if (tile_smem_bytes(e1m, e2m) <= smem_budget || (N + NT - 1) / NT <= 2) break;
    }
  }
  std::vector<int32_t> inv(N);
  for (int64_t d = 0; d < N; ++d) inv[ord[d]] = (int32_t)d;
  std::vector<double> nxP(N), nyP(N), nzP(N), fP(N), hsP(N);
  {
    std::vector<std::vector<int32_t>> colsP(N);
    std::vector<int32_t> cntP(N), dfxP(N);
    std::vector<double> coefP(coef.size()), df1P(df1.size());
    for (int64_t d = 0; d < N; ++d) {
      const int64_t i = ord[d];
      for (int32_t j : cols[i]) colsP[d].push_back(inv[j]);
      cntP[d] = cnt[i];
      dfxP[d] = dfx[i];
      for (int s2 = 0; s2 < K; ++s2) {
        for (int o = 0; o < NOPS; ++o)
          coefP[((size_t)s2 * NOPS + o) * N + d] = coef[((size_t)s2 * NOPS + o) * N + i];
        df1P[(size_t)s2 * N + d] = df1[(size_t)s2 * N + i];
        nbr[(size_t)s2 * N + d] = s2 < cntP[d] ? colsP[d][s2] : (int32_t)d;
      }
      nxP[d] = n_x[i];
      nyP[d] = n_y[i];
      nzP[d] = n_z[i];
      fP[d] = f[i];
      hsP[d] = h_s[i];
    }
    cols.swap(colsP);
    cnt.swap(cntP);
    dfx.swap(dfxP);
    coef.swap(coefP);
    df1.swap(df1P);
    n_x = nxP.data();
    n_y = nyP.data();
    n_z = nzP.data();
    f = fP.data();
    h_s = hsP.data();
  }
  // ---- compact (off-diagonal) stencil for the tiled Krylov pass, valid when
  // G, V, L rows sum to zero and D's diagonal is + the off-diagonal sum
  int KC = 1;
  std::vector<int32_t> offn((size_t)KMAX * N);
  std::vector<int32_t> offc(N);
  bool tiled_ok = true;
  for (int64_t i = 0; i < N; ++i) {
    int q = 0;
    for (int s2 = 0; s2 < cnt[i]; ++s2)
      if (cols[i][s2] != i) offn[(size_t)q++ * N + i] = cols[i][s2];
    offc[i] = q;
    KC = std::max(KC, q);
    for (int o = 0; o < NOPS && tiled_ok; ++o) {
      double off = 0.0, mag = 0.0, dg = 0.0;
      for (int s2 = 0; s2 < cnt[i]; ++s2) {
        const double v = coef[((size_t)s2 * NOPS + o) * N + i];
        if (cols[i][s2] == i) dg = v;
        else { off += v; mag += std::fabs(v); }
      }
      const double want = (o >= OP_DX && o <= OP_DZ) ? off : -off;
      if (std::fabs(dg - want) > 1e-10 * mag + 1e-300) tiled_ok = false;
    }
  }
  if (KC > KCMAX) tiled_ok = false;
  KC = std::min(KC, KCMAX);
  for (int64_t i = 0; i < N; ++i)
    for (int q = offc[i]; q < KMAX; ++q) offn[(size_t)q * N + i] = (int32_t)i;
  const int64_t NC = (N + 1) & ~(int64_t)1;  // even run stride: 16-byte aligned TMA runs
  std::vector<double> coefc((size_t)KCMAX * 9 * NC + 2, 0.0);
  std::vector<double> Lc((size_t)N * 8, 0.0);
  // compact op order: Vx Vy Vz Gx Gy Gz Dx Dy Dz
  const int corder[9] = {OP_VX, OP_VY, OP_VZ, OP_GX, OP_GY, OP_GZ, OP_DX, OP_DY, OP_DZ};
  for (int64_t i = 0; i < N; ++i) {
    int q = 0;
    for (int s2 = 0; s2 < cnt[i] && q < KC; ++s2) {
      if (cols[i][s2] == i) continue;
      for (int k = 0; k < 9; ++k)
        coefc[((size_t)q * 9 + k) * NC + i] = coef[((size_t)s2 * NOPS + corder[k]) * N + i];
      Lc[(size_t)i * 8 + q] = coef[((size_t)s2 * NOPS + OP_L) * N + i];
      ++q;
    }
  }

  std::vector<int32_t> t_cell0(NT), t_nT(NT), t_nE1(NT), t_nE2(NT), t_e2off(NT), t_e1off(NT);
  std::vector<int32_t> e2map;
  std::vector<int16_t> lnbr;
  std::vector<double> LcE1;  // Laplacian rows of every tile's E1 cells, local order
  int e1max = 1, e2max = 1;
  {
    std::vector<int32_t> loc(N, -1), list;
    bool sort_halo = false;
    if (const char* e = getenv("EIK_SORT_HALO")) sort_halo = atoi(e) != 0;
    for (int t = 0; t < NT; ++t) {
      const int64_t lo = tstart[t], hi = tstart[t + 1];
      list.clear();
      for (int64_t i = lo; i < hi; ++i) { loc[i] = (int32_t)list.size(); list.push_back((int32_t)i); }
      const int nT = (int)list.size();
      for (int64_t i = lo; i < hi; ++i)
        for (int q = 0; q < cnt[i]; ++q) {
          const int32_t j = nbr[(size_t)q * N + i];
          if (loc[j] < 0) { loc[j] = (int32_t)list.size(); list.push_back(j); }
        }
      const int nE1 = (int)list.size();
      for (int c2 = nT; c2 < nE1; ++c2) {
        const int32_t gi = list[c2];
        for (int q = 0; q < cnt[gi]; ++q) {
          const int32_t j = nbr[(size_t)q * N + gi];
          if (loc[j] < 0) { loc[j] = (int32_t)list.size(); list.push_back(j); }
        }
      }
      const int nE2 = (int)list.size();
      if (sort_halo) {
        // each halo ring in ascending device order (labels only: the stencil
        // sums keep their slot order)
        std::sort(list.begin() + nT, list.begin() + nE1);
        std::sort(list.begin() + nE1, list.end());
        for (int c2 = nT; c2 < nE2; ++c2) loc[list[c2]] = c2;
      }
      if (nE2 > 32767) return fail(EIK_EINVAL, "tile halo too large");
      t_cell0[t] = (int32_t)lo; t_nT[t] = nT; t_nE1[t] = nE1; t_nE2[t] = nE2;
      t_e2off[t] = (int32_t)e2map.size();
      t_e1off[t] = (int32_t)(lnbr.size() / 8);
      for (int c2 = 0; c2 < nE1; ++c2) {
        const int32_t gi = list[c2];
        for (int q = 0; q < 8; ++q) {
          const int32_t j = q < KMAX ? offn[(size_t)q * N + gi] : gi;
          lnbr.push_back((int16_t)loc[j]);
        }
        for (int q = 0; q < KCMAX; ++q) LcE1.push_back(Lc[(size_t)gi * 8 + q]);
      }
      for (int32_t g2 : list) { e2map.push_back(g2); loc[g2] = -1; }
      while (e2map.size() & 3) e2map.push_back(0);  // 16-byte aligned per-tile runs
      e1max = std::max(e1max, nE1);
      e2max = std::max(e2max, nE2);
    }
  }
  // ---- balance: tile t is processed by CTA t % Gt in the kernels; permute
  // the tiles so that this static assignment is a longest-processing-time
  // schedule of the per-tile cost (own cells + halo gathers), padding every
  // CTA to the same count with empty tiles
  // (measured: LPT scatters the tiles processed concurrently and loses the L2
  // locality of the halo gathers -- 182 vs 143 us per Krylov iteration at L8 --
  // so it is off; round-robin keeps every wave a contiguous range of the device order)
  int NTb = NT;
  if (EIK_LPT) {
    std::vector<double> cost(NT);
    for (int t = 0; t < NT; ++t) cost[t] = t_nT[t] + 0.6 * t_nE2[t] + 0.3 * t_nE1[t];
    std::vector<int> order(NT);
    for (int t = 0; t < NT; ++t) order[t] = t;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    std::vector<double> load(Gt, 0.0);
    std::vector<std::vector<int>> lists(Gt);
    for (int t : order) {
      int best = 0;
      for (int g2 = 1; g2 < Gt; ++g2)
        if (load[g2] < load[best]) best = g2;
      load[best] += cost[t];
      lists[best].push_back(t);
    }
    size_t per_cta = 0;
    for (auto& l : lists) per_cta = std::max(per_cta, l.size());
    NTb = (int)(per_cta * Gt);
    std::vector<int32_t> c0b(NTb, 0), nTb(NTb, 0), nE1b(NTb, 0), nE2b(NTb, 0), e2b(NTb, 0),
        e1b(NTb, 0);
    for (int g2 = 0; g2 < Gt; ++g2)
      for (size_t k2 = 0; k2 < lists[g2].size(); ++k2) {
        const int src = lists[g2][k2];
        const int dst = (int)(k2 * Gt + g2);
        c0b[dst] = t_cell0[src];
        nTb[dst] = t_nT[src];
        nE1b[dst] = t_nE1[src];
        nE2b[dst] = t_nE2[src];
        e2b[dst] = t_e2off[src];
        e1b[dst] = t_e1off[src];
      }
    t_cell0.swap(c0b);
    t_nT.swap(nTb);
    t_nE1.swap(nE1b);
    t_nE2.swap(nE2b);
    t_e2off.swap(e2b);
    t_e1off.swap(e1b);
  }
  // tile-major coefficient blocks: each tile's 54 runs contiguous (run stride
  // nT rounded up to 16 doubles, so every run starts on a 128-byte line) instead
  // of 54 global runs of N: a tile streams one ~100 KB block, not 54 2-KB pieces
  // 5 MB apart.  With EIK_FIXCS (default) the run stride is TILE for every tile.
  bool tilecoef = !EIK_LPT;
  if (!EIK_FIXCS)
    if (const char* e = getenv("EIK_TILECOEF")) tilecoef = tilecoef && atoi(e) != 0;
  std::vector<int32_t> t_coff(NTb, 0);
  if (tilecoef) {
    size_t tot = 0;
    for (int t = 0; t < NTb; ++t) {
      t_coff[t] = (int32_t)(tot / 16);
      tot += (size_t)NCOEF * (EIK_FIXCS ? TILE : ((t_nT[t] + 15) & ~15));
    }
    if (tot / 16 > (size_t)INT32_MAX) {
      tilecoef = false;
    } else {
      std::vector<double> blk(tot + 16, 0.0);
      for (int t = 0; t < NTb; ++t) {
        const size_t cs = EIK_FIXCS ? (size_t)TILE : (size_t)((t_nT[t] + 15) & ~15);
        const size_t b0 = (size_t)t_coff[t] * 16;
        for (int r = 0; r < NCOEF; ++r)
          for (int cc = 0; cc < t_nT[t]; ++cc)
            blk[b0 + r * cs + cc] = coefc[(size_t)r * NC + t_cell0[t] + cc];
      }
      coefc.swap(blk);
    }
    if (!tilecoef) std::fill(t_coff.begin(), t_coff.end(), 0);
  }
  if (EIK_FIXCS && !tilecoef)
    return fail(EIK_EINVAL, "the fixed-stride build needs the tile-major coefficient blocks");
  EikSwe* c = new EikSwe();
  c->N = N;
  c->K = K;
  c->c09cube = std::pow(0.9, 3.0);
  // the step path's engine calls use PhiTask's default m_max = 100
  // (phipm.py:87-107): the basis always holds min(100, n) vectors
  eik_status s = c->eng.init(device, N, 4 * N,
                             std::min<int64_t>(std::max<int64_t>(m_max, kStepMMax), 4 * N),
                             kSweKernels, 9, tile_smem_bytes(e1max, e2max), Gt);
  if (s != EIK_OK) { c->eng.release(); delete c; return s; }
  Bufs& B = c->eng.mem;
  int *d_nbr, *d_dfx, *d_cnt;
  double *d_coef, *d_df1, *d_hs;
  double4* d_nf;
#define CKC(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      c->eng.release();                                                        \
      delete c;                                                                \
      return fail(EIK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                          \
  } while (0)
  CKC(B.get(&d_nbr, (size_t)K * N));
  CKC(B.get(&d_coef, (size_t)K * NOPS * N));
  CKC(B.get(&d_df1, (size_t)K * N));
  CKC(B.get(&d_dfx, N));
  CKC(B.get(&d_cnt, N));
  CKC(B.get(&d_hs, N));
  CKC(B.get(&d_nf, N));
  CKC(cudaMemcpy(d_nbr, nbr.data(), nbr.size() * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_coef, coef.data(), coef.size() * 8, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_df1, df1.data(), df1.size() * 8, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_dfx, dfx.data(), dfx.size() * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_cnt, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_hs, h_s, N * 8, cudaMemcpyHostToDevice));
  int *d_tc0, *d_tnT, *d_tnE1, *d_tnE2, *d_te2, *d_te1, *d_e2map;
  short* d_lnbr;
  double* d_Lc;
  CKC(B.get(&d_tc0, NTb));
  CKC(B.get(&d_tnT, NTb));
  CKC(B.get(&d_tnE1, NTb));
  CKC(B.get(&d_tnE2, NTb));
  CKC(B.get(&d_te2, NTb));
  CKC(B.get(&d_te1, NTb));
  CKC(B.get(&d_e2map, e2map.size()));
  CKC(B.get(&d_lnbr, lnbr.size()));
  CKC(B.get(&d_Lc, Lc.size()));
  double* d_coefc;
  double* d_LcE1;
  CKC(B.get(&d_LcE1, LcE1.size() + 2));
  CKC(cudaMemcpy(d_LcE1, LcE1.data(), LcE1.size() * 8, cudaMemcpyHostToDevice));
  CKC(B.get(&d_coefc, coefc.size()));
  CKC(cudaMemcpy(d_coefc, coefc.data(), coefc.size() * 8, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_tc0, t_cell0.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_tnT, t_nT.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_tnE1, t_nE1.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_tnE2, t_nE2.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_te2, t_e2off.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_te1, t_e1off.data(), NTb * 4, cudaMemcpyHostToDevice));
  int* d_tcoff;
  CKC(B.get(&d_tcoff, NTb));
  CKC(cudaMemcpy(d_tcoff, t_coff.data(), NTb * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_e2map, e2map.data(), e2map.size() * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_lnbr, lnbr.data(), lnbr.size() * 2, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(d_Lc, Lc.data(), Lc.size() * 8, cudaMemcpyHostToDevice));
  {
    std::vector<double4> nf(N);
    for (int64_t i = 0; i < N; ++i) nf[i] = make_double4(n_x[i], n_y[i], n_z[i], f[i]);
    CKC(cudaMemcpy(d_nf, nf.data(), N * sizeof(double4), cudaMemcpyHostToDevice));
  }
  CKC(B.get(&c->u, N));
  CKC(B.get(&c->uprev, N));
  CKC(B.get(&c->fn, N));
  CKC(B.get(&c->v1, N));
  CKC(B.get(&c->va, N));
  CKC(B.get(&c->vb, N));
  CKC(B.get(&c->d2, N));
  CKC(B.get(&c->Ub, N));
  CKC(B.get(&c->ss, 1));
  for (int k = 0; k < 5; ++k) CKC(B.get(&c->W[k], N));
  CKC(B.get(&c->x, N));
  CKC(B.get(&c->out, N));
  CKC(B.get(&c->soa, 4 * N));
  CKC(B.get(&c->ord_d, N));
  CKC(cudaMemcpy(c->ord_d, ord.data(), N * 4, cudaMemcpyHostToDevice));
  c->ord_h = ord;
  double4 *ne, *lapA, *lapB, *gn;
  CKC(B.get(&ne, N));
  CKC(B.get(&gn, N));
  CKC(B.get(&lapA, N));
  CKC(B.get(&lapB, N));
  CKC(cudaEventCreate(&c->ev0));
  CKC(cudaEventCreate(&c->ev1));
  CKC(cudaEventCreate(&c->evs0));
  CKC(cudaEventCreate(&c->evs1));
#undef CKC
  SweOp& S = c->S;
  S.N = N;
  S.K = K;
  S.nbr = d_nbr;
  S.coef = d_coef;
  S.nf = d_nf;
  S.hs = d_hs;
  S.g = g;
  S.nu = nu;
  S.lin = c->u;
  S.ne = ne;
  S.lapA = lapA;
  S.lapB = lapB;
  S.gn = gn;
  S.scale = 1.0;
  S.df1 = d_df1;
  S.dfx = d_dfx;
  S.cnt = d_cnt;
  S.ntiles = NTb;
  S.t_cell0 = d_tc0;
  S.t_nT = d_tnT;
  S.t_nE1 = d_tnE1;
  S.t_nE2 = d_tnE2;
  S.t_e2off = d_te2;
  S.t_e1off = d_te1;
  S.e2map = d_e2map;
  S.lnbr = d_lnbr;
  S.Lc = d_Lc;
  S.coefc = d_coefc;
  S.NC = NC;
  S.t_coff = d_tcoff;
  S.tilecoef = tilecoef ? 1 : 0;
  S.LcE1 = d_LcE1;
  S.KC = KC;
  S.tiled_ok = tiled_ok ? 1 : 0;
  S.prof = nullptr;
  if (EIK_PROF) {
    unsigned long long* pr;
    if (B.get(&pr, 8) == cudaSuccess) S.prof = pr;
  }
  S.e1max = e1max;
  S.e2max = e2max;
  *out = c;
  return EIK_OK;
}

static void swe_destroy_now(EikSwe* c);
eik_status eik_swe_destroy(EikSwe* c) {
  if (!c) return EIK_OK;
  if (defer_destroy([c] { swe_destroy_now(c); })) return EIK_OK;
  swe_destroy_now(c);
  return EIK_OK;
}
static void swe_destroy_now(EikSwe* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->evs0) cudaEventDestroy(c->evs0);
  if (c->evs1) cudaEventDestroy(c->evs1);
  c->eng.release();
  delete c;
}

eik_status eik_swe_set_state(EikSwe* c, const double* u) {
  EIK_NO_REENTRY();
  if (!c || !u) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->u);
  if (s != EIK_OK) return s;
  CK(cudaStreamSynchronize(c->eng.st));
  return EIK_OK;
}

eik_status eik_swe_get_state(EikSwe* c, double* u) {
  EIK_NO_REENTRY();
  if (!c || !u) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  return c->d2h_cells(c->u, u);
}

eik_status eik_swe_set_prev(EikSwe* c, const double* u_prev) {
  EIK_NO_REENTRY();
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  if (!u_prev) {
    c->have_prev = false;
    return EIK_OK;
  }
  eik_status s = c->h2d_cells(u_prev, c->uprev);
  if (s != EIK_OK) return s;
  CK(cudaStreamSynchronize(c->eng.st));
  c->have_prev = true;
  return EIK_OK;
}

eik_status eik_swe_rhs(EikSwe* c, const double* u, double* out) {
  EIK_NO_REENTRY();
  if (!c || !u || !out) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->x);
  if (s != EIK_OK) return s;
  SweArgs A = c->args(c->x);
  if ((s = c->launch((const void*)k_swe_rhs, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  return c->d2h_cells(c->out, out);
}

eik_status eik_swe_jv(EikSwe* c, const double* u, const double* v, double* out) {
  EIK_NO_REENTRY();
  if (!c || !u || !v || !out) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->x);
  if (s == EIK_OK) s = c->h2d_cells(v, c->va);
  if (s != EIK_OK) return s;
  SweArgs A = c->args(c->x);
  if ((s = c->launch((const void*)k_swe_jv, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  return c->d2h_cells(c->out, out);
}

eik_status eik_swe_jac_nnz_rows(EikSwe* c, const double* u, int64_t* nnz,
                                double* per_cell) {
  EIK_NO_REENTRY();
  if (!c || !u || !nnz) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->x);
  if (s != EIK_OK) return s;
  SweArgs A = c->args(c->x);
  A.dbg = per_cell ? c->soa : nullptr;
  if ((s = c->launch((const void*)k_swe_nnz, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  double v = 0.0;
  CK(cudaMemcpy(&v, c->eng.nnz_d, sizeof(double), cudaMemcpyDeviceToHost));
  *nnz = (int64_t)v;
  if (per_cell) {
    std::vector<double> tmp(c->N);
    CK(cudaMemcpy(tmp.data(), c->soa, c->N * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t d = 0; d < c->N; ++d) per_cell[c->ord_h[d]] = tmp[d];
  }
  return EIK_OK;
}

eik_status eik_swe_jac_nnz(EikSwe* c, const double* u, int64_t* nnz) {
  EIK_NO_REENTRY();
  if (!c || !u || !nnz) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->x);
  if (s != EIK_OK) return s;
  SweArgs A = c->args(c->x);
  if ((s = c->launch((const void*)k_swe_nnz, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  double v = 0.0;
  CK(cudaMemcpy(&v, c->eng.nnz_d, sizeof(double), cudaMemcpyDeviceToHost));
  *nnz = (int64_t)v;
  return EIK_OK;
}

eik_status eik_swe_phipm(EikSwe* c, const double* u_lin, double dt,
                         const EikPhiTask* task, double* W, EikPhipmInfo* info,
                         EikTraceRec* trace, int64_t trace_cap, int64_t* trace_len) {
  EIK_NO_REENTRY();
  if (!c || !u_lin || !W) return fail(EIK_EINVAL, "invalid arguments");
  EngineHost& E = c->eng;
  if (task && task->m_max > E.m_alloc) {
    // a larger m_max than the context was created for: grow the basis (the
    // cached step graph holds the old pointers)
    eik_status r = E.reserve(task->m_max);
    if (r != EIK_OK) return r;
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
      c->g_scheme = -1;
    }
  }
  eik_status s = E.check_task(task);
  if (s != EIK_OK) return s;
  CK(cudaSetDevice(E.dev));
  if ((s = E.ensure_io()) != EIK_OK) return s;
  if ((s = c->h2d_cells(u_lin, c->x)) != EIK_OK) return s;
  for (int l = 0; l <= task->p; ++l)
    if (task->v && task->v[l] && (s = c->h2d_cells(task->v[l], E.vin[l])) != EIK_OK) return s;
  if (trace && trace_cap > 0 && (s = E.ensure_trace(trace_cap)) != EIK_OK) return s;
  SweArgs A = c->args(c->x, dt);
  A.dt = dt;
  A.task = E.make_task(task);
  A.Wk.trace = (trace && trace_cap > 0) ? E.trace_d : nullptr;
  A.Wk.trace_cap = (trace && trace_cap > 0) ? trace_cap : 0;
  CK(cudaMemsetAsync(E.trace_len_d, 0, sizeof(int64_t), E.st));
  CK(cudaEventRecord(c->ev0, E.st));
  if ((s = c->launch((const void*)k_swe_phipm, A)) != EIK_OK) return s;
  CK(cudaEventRecord(c->ev1, E.st));
  s = E.finish_phipm(info, trace, trace_cap, trace_len);
  cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
  if (s != EIK_OK) return s;
  for (int i = 0; i < task->ns; ++i)
    if ((s = c->d2h_cells(E.wout[i], W + (size_t)i * 4 * c->N)) != EIK_OK) return s;
  return EIK_OK;
}

// The step graph.  Split (default):  k_swe_cont ; while (cond) { k_swe_sweep ;
// k_swe_cont }  with the loop condition set on the device.  Monolithic
// (EIK_STEP_MONO=1, or when the conditional graph cannot be built): one
// k_swe_step launch.
struct GraphLaunch {
  const void* fn;
  SweArgs* args;
  bool coop;
  int grid, block;
  size_t smem;
};

static bool dense_attr_set() {
  static bool done = false;
  if (!done)
    done = cudaFuncSetAttribute((const void*)k_swe_dense,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kDenseKernelSmem) == cudaSuccess;
  return done;
}

static bool capture_launches(cudaStream_t st, cudaGraph_t g, const GraphLaunch* L, int nk) {
  if (cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return false;
  bool ok = true;
  for (int k = 0; k < nk && ok; ++k) {
    void* kargs[] = {L[k].args};
    ok = (L[k].coop ? cudaLaunchCooperativeKernel(L[k].fn, L[k].grid, L[k].block, kargs,
                                                  L[k].smem, st)
                    : cudaLaunchKernel(L[k].fn, L[k].grid, L[k].block, kargs, L[k].smem, st)) ==
         cudaSuccess;
  }
  cudaGraph_t out = g;
  ok = (cudaStreamEndCapture(st, &out) == cudaSuccess) && ok;
  return ok;
}

static bool build_step_graph(EikSwe* c, const SweArgs& A, bool split, cudaGraphExec_t* exec) {
  cudaGraph_t g = nullptr;
  bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
  if (ok && !split) {
    SweArgs A0 = A;
    const GraphLaunch L0[] = {{(const void*)k_swe_step, &A0, true, c->eng.G, TPB, c->eng.smem}};
    ok = capture_launches(c->eng.st, g, L0, 1);
  } else if (ok) {
    cudaGraphConditionalHandle h = 0;
    ok = cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) == cudaSuccess;
    SweArgs A0 = A, A1 = A;
    A0.cond = A1.cond = h;
    A0.resume = 0;
    A1.resume = 1;
    const int G = c->eng.G;
    const size_t sm = c->eng.smem;
    const GraphLaunch L0[] = {{(const void*)k_swe_cont, &A0, true, G, TPB, sm}};
    const GraphLaunch L1[] = {{(const void*)k_swe_sweep, &A1, true, G, TPB, sm},
                              {(const void*)k_swe_dense, &A1, false, 1, kDenseNT, kDenseKernelSmem},
                              {(const void*)k_swe_cont, &A1, true, G, TPB, sm}};
    ok = ok && dense_attr_set();
    ok = ok && capture_launches(c->eng.st, g, L0, 1);
    cudaGraphNode_t first = nullptr;
    size_t nn = 1;
    ok = ok && cudaGraphGetNodes(g, &first, &nn) == cudaSuccess && nn == 1;
    alignas(cudaGraphNodeParams) unsigned char cp_raw[sizeof(cudaGraphNodeParams)] = {};
    cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_raw);
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn = nullptr;
    ok = ok && cudaGraphAddNode(&cn, g, &first, 1, &cp) == cudaSuccess;
    ok = ok && capture_launches(c->eng.st, cp.conditional.phGraph_out[0], L1, 3);
  }
  ok = ok && cudaGraphInstantiate(exec, g, 0) == cudaSuccess;
  if (g) cudaGraphDestroy(g);
  if (!ok) {
    cudaGetLastError();
    *exec = nullptr;
  }
  return ok;
}

// The split step without a graph: cont ; while (ss->more) { sweep ; dense ; cont }.
static eik_status step_hostloop(EikSwe* c, SweArgs A) {
  if (!dense_attr_set()) return fail(EIK_ECUDA, "k_swe_dense shared-memory attribute");
  A.hostloop = 1;
  A.cond = 0;
  A.resume = 0;
  if (c->sweep_log)
    CK(cudaMemcpy(&c->kit_last, c->eng.kiters_d, sizeof(c->kit_last), cudaMemcpyDeviceToHost));
  // (launch counts: these kernels count themselves on the device)
  void* kargs[] = {&A};
  const int G = c->eng.G;
  const size_t sm = c->eng.smem;
  CK(cudaLaunchCooperativeKernel((const void*)k_swe_cont, G, TPB, kargs, sm, c->eng.st));
  A.resume = 1;
  for (;;) {
    int more = 0;
    CK(cudaMemcpyAsync(&more, &c->ss->more, sizeof(int), cudaMemcpyDeviceToHost, c->eng.st));
    CK(cudaStreamSynchronize(c->eng.st));
    if (!more) break;
    CK(cudaEventRecord(c->evs0, c->eng.st));
    CK(cudaLaunchCooperativeKernel((const void*)k_swe_sweep, G, TPB, kargs, sm, c->eng.st));
    CK(cudaEventRecord(c->evs1, c->eng.st));
    CK(cudaLaunchKernel((const void*)k_swe_dense, 1, kDenseNT, kargs, kDenseKernelSmem,
                        c->eng.st));
    CK(cudaLaunchCooperativeKernel((const void*)k_swe_cont, G, TPB, kargs, sm, c->eng.st));
    CK(cudaEventSynchronize(c->evs1));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, c->evs0, c->evs1));
    c->sweep_ms += ms;
    if (c->sweep_log) {
      // per-sweep record for matching ncu captures (launch index, iterations)
      unsigned long long kit = 0;
      CK(cudaMemcpy(&kit, c->eng.kiters_d, sizeof(kit), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[eik] sweep %lld iters %llu ms %.4f\n", (long long)c->nsweeps,
              kit - c->kit_last, ms);
      c->kit_last = kit;
    }
    ++c->nsweeps;
  }
  return EIK_OK;
}

static eik_status step_enqueue(EikSwe* c, int32_t scheme, double dt, double tol) {
  SweArgs A = c->args(c->u, dt);
  A.dt = dt;
  A.tol = tol;
  A.scheme = scheme;
  A.ss = c->ss;
  if (c->hostloop) return step_hostloop(c, A);
  if (c->graphs_ok) {
    if (!c->gexec || c->g_scheme != scheme || c->g_dt != dt || c->g_tol != tol) {
      if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
      }
      if (c->split && !build_step_graph(c, A, true, &c->gexec)) c->split = false;
      if (!c->split && !build_step_graph(c, A, false, &c->gexec)) c->graphs_ok = false;
      if (c->gexec) {
        c->g_scheme = scheme;
        c->g_dt = dt;
        c->g_tol = tol;
      }
    }
    if (c->graphs_ok) {
      CK(cudaGraphLaunch(c->gexec, c->eng.st));
      if (!c->split) ++c->eng.launches;  // split: kernels are counted on the device
      return EIK_OK;
    }
  }
  return c->launch((const void*)k_swe_step, A);
}

eik_status eik_swe_step(EikSwe* c, int32_t scheme, double dt, double tol,
                        EikPhipmInfo* calls, int32_t* ncalls) {
  EIK_NO_REENTRY();
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  if (!(dt > 0.0)) return fail(EIK_EINVAL, "dt must be positive");
  if (scheme < 0 || scheme > EIK_EXPRB53) return fail(EIK_EINVAL, "unknown scheme");
  if (scheme == EIK_EPI3 && !c->have_prev)
    return fail(EIK_EINVAL, "epi3 requires the previous state");
  CK(cudaSetDevice(c->eng.dev));
  CK(cudaEventRecord(c->ev0, c->eng.st));
  eik_status s = step_enqueue(c, scheme, dt, tol);
  if (s != EIK_OK) return s;
  CK(cudaEventRecord(c->ev1, c->eng.st));
  EikPhipmInfo inf[4];
  CK(cudaMemcpyAsync(inf, c->eng.info_d, sizeof(inf), cudaMemcpyDeviceToHost, c->eng.st));
  s = c->status();
  cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
  const int nc = scheme == EIK_EXPRB53 ? 3 : (scheme >= EIK_EXPRB42 ? 2 : 1);
  if (calls)
    for (int k = 0; k < nc; ++k) calls[k] = inf[k];
  if (ncalls) *ncalls = nc;
  if (s == EIK_OK) c->have_prev = true;
  return s;
}

eik_status eik_swe_advance(EikSwe* c, int32_t scheme, double dt, double tol,
                           int32_t nsteps, int64_t* matvecs, int64_t* substeps) {
  EIK_NO_REENTRY();
  if (!c || nsteps < 0) return fail(EIK_EINVAL, "invalid arguments");
  if (scheme == EIK_EPI3 && !c->have_prev)
    return fail(EIK_EINVAL, "epi3 requires the previous state");
  int64_t mv = 0, ss = 0;
  for (int k = 0; k < nsteps; ++k) {
    EikPhipmInfo calls[3];
    int32_t nc = 0;
    eik_status s = eik_swe_step(c, scheme, dt, tol, calls, &nc);
    if (s != EIK_OK) return s;
    for (int q = 0; q < nc; ++q) {
      mv += calls[q].matvecs;
      ss += calls[q].substeps;
    }
  }
  if (matvecs) *matvecs = mv;
  if (substeps) *substeps = ss;
  return EIK_OK;
}

eik_status eik_swe_seeds(EikSwe* c, int32_t slot, double* tau, int64_t* m, int32_t set) {
  if (!c || slot < 0 || slot >= EIK_NUM_SLOTS || !tau || !m)
    return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  double v[2];
  if (set) {
    v[0] = *tau > 0.0 ? *tau : -1.0;
    v[1] = (double)*m;
    CK(cudaMemcpy(c->eng.wk.seeds + 2 * slot, v, sizeof(v), cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemcpy(v, c->eng.wk.seeds + 2 * slot, sizeof(v), cudaMemcpyDeviceToHost));
    *tau = v[0];
    *m = (int64_t)v[1];
  }
  return EIK_OK;
}

eik_status eik_swe_reset_seeds(EikSwe* c) {
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  return c->eng.reset_seeds();
}

eik_status eik_swe_snapshot(EikSwe* c, int32_t restore) {
  EIK_NO_REENTRY();
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  const size_t vb = (size_t)c->N * sizeof(double4), sb = 2 * EIK_NUM_SLOTS * sizeof(double);
  if (!c->snap_u) {
    if (restore) return fail(EIK_EINVAL, "no snapshot taken");
    CK(c->eng.mem.get(&c->snap_u, c->N));
    CK(c->eng.mem.get(&c->snap_prev, c->N));
    CK(c->eng.mem.get(&c->snap_seeds, 2 * EIK_NUM_SLOTS));
  }
  cudaStream_t st = c->eng.st;
  if (restore) {
    CK(cudaMemcpyAsync(c->u, c->snap_u, vb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->uprev, c->snap_prev, vb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->eng.wk.seeds, c->snap_seeds, sb, cudaMemcpyDeviceToDevice, st));
    c->have_prev = c->snap_have_prev;
  } else {
    CK(cudaMemcpyAsync(c->snap_u, c->u, vb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->snap_prev, c->uprev, vb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->snap_seeds, c->eng.wk.seeds, sb, cudaMemcpyDeviceToDevice, st));
    c->snap_have_prev = c->have_prev;
  }
  return EIK_OK;
}


eik_status eik_swe_krylov_bench(EikSwe* c, const double* u, const double* v, double dt,
                                int32_t m, int32_t reps, double* out) {
  EIK_NO_REENTRY();
  if (!c || !u || !v || !out || m < 1 || reps < 1) return fail(EIK_EINVAL, "invalid arguments");
  if (m > c->eng.m_alloc) return fail(EIK_EINVAL, "m exceeds the basis allocation");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = c->h2d_cells(u, c->x);
  if (s == EIK_OK) s = c->h2d_cells(v, c->va);
  if (s != EIK_OK) return s;
  SweArgs A = c->args(c->x, dt);
  A.dt = dt;
  A.scheme = m;
  A.tol = 1.0;  // warm-up launch: one sweep
  if ((s = c->launch((const void*)k_swe_kbench, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  A.tol = (double)reps;
  CK(cudaEventRecord(c->ev0, c->eng.st));
  if ((s = c->launch((const void*)k_swe_kbench, A)) != EIK_OK) return s;
  CK(cudaEventRecord(c->ev1, c->eng.st));
  if ((s = c->status()) != EIK_OK) return s;
  float ms = 0.0f;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  double keep = 0.0;
  CK(cudaMemcpy(&keep, c->eng.nnz_d, sizeof(double), cudaMemcpyDeviceToHost));
  out[0] = ms;
  out[1] = keep;
  return EIK_OK;
}


eik_status eik_swe_diagnostics(EikSwe* c, const double* u, const double* weights,
                               double cell_area, double* out) {
  EIK_NO_REENTRY();
  if (!c || !out) return fail(EIK_EINVAL, "invalid arguments");
  CK(cudaSetDevice(c->eng.dev));
  eik_status s = EIK_OK;
  double4* src = c->u;
  if (u) {
    if ((s = c->h2d_cells(u, c->x)) != EIK_OK) return s;
    src = c->x;
  }
  double* wdev = nullptr;
  if (weights) {
    if (!c->wts) CK(c->eng.mem.get(&c->wts, c->N));
    std::vector<double> wp(c->N);
    for (int64_t d = 0; d < c->N; ++d) wp[d] = weights[c->ord_h[d]];
    CK(cudaMemcpyAsync(c->wts, wp.data(), c->N * sizeof(double), cudaMemcpyHostToDevice,
                       c->eng.st));
    CK(cudaStreamSynchronize(c->eng.st));
    wdev = c->wts;
  }
  SweArgs A = c->args(src);
  A.x = src;
  A.dbg = wdev;
  A.tol = cell_area;
  if ((s = c->launch((const void*)k_swe_diag, A)) != EIK_OK) return s;
  if ((s = c->status()) != EIK_OK) return s;
  double v[4];
  CK(cudaMemcpy(v, c->eng.nnz_d, sizeof(v), cudaMemcpyDeviceToHost));
  if (v[3] > 0.0) return fail(EIK_EINVAL, "height field must be positive");
  out[0] = v[0];
  out[1] = v[1];
  out[2] = v[2];
  return EIK_OK;
}

eik_status eik_swe_info(const EikSwe* c, int64_t* out) {
  if (!c || !out) return fail(EIK_EINVAL, "invalid arguments");
  out[0] = c->eng.G;
  out[1] = TPB;
  out[2] = c->S.ntiles;
  out[3] = c->S.e1max;
  out[4] = c->S.e2max;
  out[5] = c->S.K;
  out[6] = c->S.KC;
  out[7] = c->S.tiled_ok;
  out[8] = (int64_t)c->eng.smem;
  if (c->S.prof) {
    unsigned long long pv[5];
    cudaMemcpy(pv, c->S.prof, sizeof(pv), cudaMemcpyDeviceToHost);
    for (int k = 0; k < 5; ++k) out[9 + k] = (int64_t)pv[k];
  }
  return EIK_OK;
}

int eik_prof_read(double* out, int reset) {
  unsigned long long v[PC_N];
  if (cudaMemcpyFromSymbol(v, g_prof, sizeof(v)) != cudaSuccess) return EIK_ECUDA;
  for (int k = 0; k < PC_N; ++k) out[k] = (double)v[k];
  if (reset) {
    memset(v, 0, sizeof(v));
    if (cudaMemcpyToSymbol(g_prof, v, sizeof(v)) != cudaSuccess) return EIK_ECUDA;
  }
  return EIK_PROF ? EIK_OK : EIK_EINVAL;
}

int64_t eik_swe_launches(const EikSwe* c) {
  if (!c) return 0;
  unsigned long long v[3] = {0, 0, 0};  // [2]: split-step kernels, counted on the device
  cudaMemcpy(v, c->eng.kiters_d, sizeof(v), cudaMemcpyDeviceToHost);
  return c->eng.launches + (int64_t)v[2];
}
double eik_swe_last_kernel_ms(const EikSwe* c) { return c ? (double)c->last_ms : 0.0; }
eik_status eik_swe_set_hostloop(EikSwe* c, int32_t on) {
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  c->hostloop = on != 0;
  return EIK_OK;
}
eik_status eik_swe_sweep_timing(EikSwe* c, double* ms, int64_t* nsweeps, int32_t reset) {
  if (!c) return fail(EIK_EINVAL, "invalid arguments");
  if (ms) *ms = c->sweep_ms;
  if (nsweeps) *nsweeps = c->nsweeps;
  if (reset) {
    c->sweep_ms = 0.0;
    c->nsweeps = 0;
  }
  return EIK_OK;
}
int64_t eik_swe_krylov_iters(const EikSwe* c) {
  if (!c) return 0;
  unsigned long long v = 0;
  cudaMemcpy(&v, c->eng.kiters_d, sizeof(v), cudaMemcpyDeviceToHost);
  return (int64_t)v;
}

int64_t eik_swe_explicit_orth(const EikSwe* c) {
  if (!c) return 0;
  unsigned long long v[2] = {0, 0};
  cudaMemcpy(v, c->eng.kiters_d, sizeof(v), cudaMemcpyDeviceToHost);
  return (int64_t)v[1];
}

// ------------------------------------------------------------------ CSR
eik_status eik_csr_create(int32_t n, EikCsrView A, int32_t device, int32_t m_max,
                          EikCsr** out) {
  EIK_NO_REENTRY();
  if (!out || n < 1 || !A.indptr || A.indptr[n] != A.nnz)
    return fail(EIK_EINVAL, "invalid CSR operator");
  for (int64_t k = 0; k < A.nnz; ++k) {
    if (A.indices[k] < 0 || A.indices[k] >= n) return fail(EIK_EINVAL, "column index out of range");
    if (!std::isfinite(A.data[k])) return fail(EIK_EINVAL, "SparseMatrix entries must be finite");
  }
  EikCsr* c = new EikCsr();
  const int64_t NU = (n + 3) / 4;
  eik_status s = c->eng.init(device, NU, n,
                             std::min<int64_t>(std::min<int64_t>(std::max(m_max, 1), n), MAXDIM),
                             kCsrKernels, 1, kDenseSmemBytes);
  if (s != EIK_OK) { c->eng.release(); delete c; return s; }
  int *rp, *ci;
  double* val;
  Bufs& B = c->eng.mem;
  if (B.get(&rp, n + 1) != cudaSuccess || B.get(&ci, std::max<int64_t>(A.nnz, 1)) != cudaSuccess ||
      B.get(&val, std::max<int64_t>(A.nnz, 1)) != cudaSuccess) {
    c->eng.release();
    delete c;
    return fail(EIK_ENOMEM, "device allocation failed");
  }
  cudaMemcpy(rp, A.indptr, (n + 1) * 4, cudaMemcpyHostToDevice);
  if (A.nnz) {
    cudaMemcpy(ci, A.indices, A.nnz * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(val, A.data, A.nnz * 8, cudaMemcpyHostToDevice);
  }
  c->C.n = n;
  c->C.NUu = NU;
  c->C.rp = rp;
  c->C.ci = ci;
  c->C.val = val;
  c->C.scale = 1.0;
  c->nnz = A.nnz;
  *out = c;
  return EIK_OK;
}

eik_status eik_csr_destroy(EikCsr* c) {
  if (!c) return EIK_OK;
  auto now = [c] {
    c->eng.release();
    delete c;
  };
  if (!defer_destroy(now)) now();
  return EIK_OK;
}

eik_status eik_csr_phipm(EikCsr* c, double scale, int64_t nnz_override,
                         const EikPhiTask* task, double* W, EikPhipmInfo* info,
                         EikTraceRec* trace, int64_t trace_cap, int64_t* trace_len) {
  EIK_NO_REENTRY();
  if (!c || !W) return fail(EIK_EINVAL, "invalid arguments");
  EngineHost& E = c->eng;
  if (task && task->m_max > E.m_alloc) {
    eik_status r = E.reserve(task->m_max);
    if (r != EIK_OK) return r;
  }
  eik_status s = E.check_task(task);
  if (s != EIK_OK) return s;
  CK(cudaSetDevice(E.dev));
  if ((s = E.ensure_io()) != EIK_OK) return s;
  const int64_t n = E.n;
  for (int l = 0; l <= task->p; ++l) {
    CK(cudaMemsetAsync(E.vin[l], 0, E.NU * sizeof(double4), E.st));
    if (task->v && task->v[l])
      CK(cudaMemcpyAsync(E.vin[l], task->v[l], n * sizeof(double), cudaMemcpyHostToDevice, E.st));
  }
  if (trace && trace_cap > 0 && (s = E.ensure_trace(trace_cap)) != EIK_OK) return s;
  CsrArgs A;
  memset(&A, 0, sizeof(A));
  A.C = c->C;
  A.C.scale = scale;
  A.Wk = E.wk;
  A.Wk.nnz = nnz_override >= 0 ? nnz_override : c->nnz;
  A.Wk.trace = (trace && trace_cap > 0) ? E.trace_d : nullptr;
  A.Wk.trace_cap = (trace && trace_cap > 0) ? trace_cap : 0;
  A.task = E.make_task(task);
  A.status = E.status_d;
  CK(cudaMemsetAsync(E.trace_len_d, 0, sizeof(int64_t), E.st));
  void* kargs[] = {&A};
  CK(cudaLaunchCooperativeKernel((const void*)k_csr_phipm, E.G, TPB, kargs, E.smem, E.st));
  ++E.launches;
  s = E.finish_phipm(info, trace, trace_cap, trace_len);
  if (s != EIK_OK) return s;
  for (int i = 0; i < task->ns; ++i)
    CK(cudaMemcpyAsync(W + (size_t)i * n, E.wout[i], n * sizeof(double), cudaMemcpyDeviceToHost, E.st));
  CK(cudaStreamSynchronize(E.st));
  return EIK_OK;
}

// ------------------------------------------------- host-callback operator
eik_status eik_cb_create(int64_t n, int32_t device, int32_t m_max, EikCb** out) {
  EIK_NO_REENTRY();
  if (!out || n < 1) return fail(EIK_EINVAL, "invalid arguments");
  EikCb* c = new EikCb();
  const int64_t NU = (n + 3) / 4;
  eik_status s = c->eng.init(device, NU, n,
                             std::min<int64_t>(std::min<int64_t>(std::max(m_max, 1), n), MAXDIM),
                             kCbKernels, 1, kDenseSmemBytes);
  auto bail = [&](eik_status st, const char* msg) {
    if (c->xh) cudaFreeHost(c->xh);
    if (c->yh) cudaFreeHost(c->yh);
    if (c->mbox) cudaFreeHost(c->mbox);
    if (c->cst) cudaStreamDestroy(c->cst);
    c->eng.release();
    delete c;
    return fail(st, msg);
  };
  if (s != EIK_OK) return bail(s, "engine init failed");
  if (cudaHostAlloc((void**)&c->xh, n * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->yh, n * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->mbox, 64, cudaHostAllocMapped) != cudaSuccess)
    return bail(EIK_ENOMEM, "pinned host allocation failed");
  if (cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess)
    return bail(EIK_ECUDA, "copy stream");
  HostOp& H = c->H;
  H.n = n;
  H.NUu = NU;
  double *xd, *yd;
  if (cudaHostGetDevicePointer((void**)&H.mbox, c->mbox, 0) != cudaSuccess)
    return bail(EIK_ECUDA, "mapped host pointer unavailable");
  if (c->eng.mem.get(&H.ctr, 2) != cudaSuccess || c->eng.mem.get(&H.abort, 1) != cudaSuccess ||
      c->eng.mem.get(&xd, 4 * NU) != cudaSuccess || c->eng.mem.get(&yd, 4 * NU) != cudaSuccess)
    return bail(EIK_ENOMEM, "device allocation failed");
  H.xh = xd;
  H.yh = yd;
  H.scale = 1.0;
  *out = c;
  return EIK_OK;
}

eik_status eik_cb_destroy(EikCb* c) {
  if (!c) return EIK_OK;
  auto now = [c] {
    cudaFreeHost(c->xh);
    cudaFreeHost(c->yh);
    cudaFreeHost(c->mbox);
    if (c->cst) cudaStreamDestroy(c->cst);
    c->eng.release();
    delete c;
  };
  if (!defer_destroy(now)) now();
  return EIK_OK;
}

eik_status eik_cb_phipm(EikCb* c, eik_matvec_fn matvec, void* user, double scale, int64_t nnz,
                        const EikPhiTask* task, double* W, EikPhipmInfo* info,
                        EikTraceRec* trace, int64_t trace_cap, int64_t* trace_len) {
  EIK_NO_REENTRY();
  if (!c || !W || !matvec) return fail(EIK_EINVAL, "invalid arguments");
  EngineHost& E = c->eng;
  if (task && task->m_max > E.m_alloc) {
    eik_status r = E.reserve(task->m_max);
    if (r != EIK_OK) return r;
  }
  eik_status s = E.check_task(task);
  if (s != EIK_OK) return s;
  CK(cudaSetDevice(E.dev));
  if ((s = E.ensure_io()) != EIK_OK) return s;
  const int64_t n = E.n;
  for (int l = 0; l <= task->p; ++l) {
    CK(cudaMemsetAsync(E.vin[l], 0, E.NU * sizeof(double4), E.st));
    if (task->v && task->v[l])
      CK(cudaMemcpyAsync(E.vin[l], task->v[l], n * sizeof(double), cudaMemcpyHostToDevice, E.st));
  }
  if (trace && trace_cap > 0 && (s = E.ensure_trace(trace_cap)) != EIK_OK) return s;
  CbArgs A;
  memset(&A, 0, sizeof(A));
  A.H = c->H;
  A.H.scale = scale;
  A.H.timeout_ns = kCbTimeoutNs;
  if (const char* e = getenv("EIK_CB_TIMEOUT_S")) {
    const double sec = atof(e);
    if (sec > 0.0) A.H.timeout_ns = (unsigned long long)(sec * 1e9);
  }
  A.Wk = E.wk;
  A.Wk.nnz = nnz;
  A.Wk.trace = (trace && trace_cap > 0) ? E.trace_d : nullptr;
  A.Wk.trace_cap = (trace && trace_cap > 0) ? trace_cap : 0;
  A.task = E.make_task(task);
  A.status = E.status_d;
  volatile unsigned int* mb = c->mbox;
  mb[0] = 0;
  mb[1] = 0;
  CK(cudaMemsetAsync(c->H.ctr, 0, 2 * sizeof(unsigned long long), E.st));
  CK(cudaMemsetAsync(c->H.abort, 0, sizeof(int), E.st));
  CK(cudaMemsetAsync(E.trace_len_d, 0, sizeof(int64_t), E.st));
  void* kargs[] = {&A};
  // destroys requested while the engine waits for the host are deferred (see g_cb_inflight)
  struct Inflight {
    Inflight() { ++g_cb_inflight; }
    ~Inflight() {
      --g_cb_inflight;
      drain_deferred();
    }
  } inflight;
  CK(cudaLaunchCooperativeKernel((const void*)k_cb_phipm, E.G, TPB, kargs, E.smem, E.st));
  ++E.launches;
  // serve the kernel's matvec requests until it finishes
  unsigned int served = 0;
  bool cb_failed = false;
  for (;;) {
    const unsigned int req = mb[0];
    if (req != served) {
      int rc = 1;
      if (!cb_failed &&
          cudaMemcpyAsync(c->xh, c->H.xh, n * sizeof(double), cudaMemcpyDeviceToHost, c->cst) ==
              cudaSuccess &&
          cudaStreamSynchronize(c->cst) == cudaSuccess) {
        g_in_callback = true;
        rc = matvec(user, c->xh, c->yh, n);
        g_in_callback = false;
        if (rc == 0 &&
            (cudaMemcpyAsync((void*)c->H.yh, c->yh, n * sizeof(double), cudaMemcpyHostToDevice,
                             c->cst) != cudaSuccess ||
             cudaStreamSynchronize(c->cst) != cudaSuccess))
          rc = 1;
      }
      if (rc != 0) cb_failed = true;
      std::atomic_thread_fence(std::memory_order_seq_cst);
      mb[1] = rc == 0 ? req : kCbAbort;
      served = req;
      continue;
    }
    const cudaError_t q = cudaStreamQuery(E.st);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return fail(EIK_ECUDA, cudaGetErrorString(q));
  }
  s = E.finish_phipm(info, trace, trace_cap, trace_len);
  if (cb_failed) return fail(EIK_ECALLBACK, "matvec callback failed");
  // a request the host did not answer in time aborts the engine on the device
  // side; an attempt already under way may still have completed on zero products
  int aborted = 0;
  CK(cudaMemcpy(&aborted, c->H.abort, sizeof(int), cudaMemcpyDeviceToHost));
  if (aborted)
    return fail(EIK_ECALLBACK, "matvec request timed out: the host did not answer (a call that "
                               "synchronises the device inside the callable?)");
  if (s != EIK_OK) return s;
  for (int i = 0; i < task->ns; ++i)
    CK(cudaMemcpyAsync(W + (size_t)i * n, E.wout[i], n * sizeof(double), cudaMemcpyDeviceToHost, E.st));
  CK(cudaStreamSynchronize(E.st));
  return EIK_OK;
}

}  // extern "C"
