/* eik.h -- C ABI of libeik.so, the B200 (sm_100a) implementation of the
 * arXiv 1805.02144 hot path: phipm_simul_iom2 (IOM2 Krylov phi-function
 * engine) + the shallow-water F(u) and J*v it drives, and the exponential
 * Rosenbrock steps EXPRB4 / pEXPRB4 / EXPRB5 and EPI3.
 *
 * Every entry point takes plain host pointers and sizes; device memory,
 * the CUDA stream and the warm-start seeds are owned by an opaque context.
 * Host buffers are borrowed only for the duration of a call.  Calls on one
 * context are serialised (the reference trajectory is sequential,
 * SPEC.md:333-334); different contexts may be used from different threads.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/expintkit):
 *   eik_swe_create      swe.DiscreteOperators          swe.py:23-46
 *   eik_swe_rhs         swe.rhs                        swe.py:149-168
 *   eik_swe_jv          assemble_jacobian(..).matvec   swe.py:220-223, kernels.py:81-82
 *   eik_swe_jac_nnz     assemble_jacobian(..).nnz      swe.py:220-223
 *   eik_swe_phipm       phipm.phipm_simul_iom2 with A = dt*J(u)
 *                                                      phipm.py:291-370, integrators.py:115-117
 *   eik_swe_step        integrators.step_{rb_euler,epi3,exprb42,pexprb43,exprb53}
 *                                                      integrators.py:140-224
 *   eik_swe_seeds       integrators.EngineSeeds        integrators.py:73-83
 *   eik_csr_phipm       phipm.phipm_simul_iom2 with A a SparseMatrix / scipy
 *                       matrix / ndarray (as_operator) phipm.py:73-84, 291-370
 */
#ifndef EIK_H
#define EIK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EIK_OK = 0,
  EIK_EINVAL = 1,      /* -> ValueError (invalid task / arguments)          */
  EIK_ENONFINITE = 2,  /* -> ValueError ("non-finite right-hand side")      */
  EIK_EPHIPM = 3,      /* -> PhipmFailure (substep budget exhausted)        */
  EIK_ECUDA = 4,       /* -> RuntimeError                                   */
  EIK_ENOMEM = 5,      /* -> MemoryError                                    */
  EIK_ECALLBACK = 6    /* host matvec callback failed: its exception re-raised */
} eik_status;

/* schemes (integrators.py:20 SCHEME_NAMES order) */
enum { EIK_RB_EULER = 0, EIK_EPI3 = 1, EIK_EXPRB42 = 2, EIK_PEXPRB43 = 3,
       EIK_EXPRB53 = 4 };

/* engine warm-start slots (integrators.py:144-222 slot names) */
enum { EIK_SLOT_RBE = 0, EIK_SLOT_EPI3 = 1, EIK_SLOT_EXPRB42_1 = 2,
       EIK_SLOT_EXPRB42_2 = 3, EIK_SLOT_PEXPRB43_1 = 4, EIK_SLOT_PEXPRB43_2 = 5,
       EIK_SLOT_EXPRB53_1 = 6, EIK_SLOT_EXPRB53_2 = 7, EIK_SLOT_EXPRB53_3 = 8,
       EIK_NUM_SLOTS = 9 };

typedef struct EikSwe EikSwe;
typedef struct EikCsr EikCsr;

/* one CSR matrix (SparseMatrix.row_offsets / col_indices / values) */
typedef struct {
  int64_t nnz;
  const int32_t* indptr;   /* n_rows + 1 */
  const int32_t* indices;  /* nnz */
  const double* data;      /* nnz */
} EikCsrView;

/* PhiTask (phipm.py:87-125).  v[l] == NULL means an all-zero vector. */
typedef struct {
  int32_t p;
  const double* const* v;  /* p+1 host pointers, each n doubles */
  int32_t ns;
  const double* rho;       /* ns strictly ascending points in (0,1] */
  double tol;
  int32_t m_init;
  int32_t iom;
  int32_t m_max;
  double delta;
  double tau_init;         /* <= 0 : None */
  int32_t zero_skip;
  int64_t max_attempts;    /* MAX_SUBSTEPS (phipm.py:28); <= 0 : 10**6 */
} EikPhiTask;

/* PhipmResult counters (phipm.py:140-148) + PhipmFailure fields */
typedef struct {
  int64_t substeps;
  int64_t rejections;
  int64_t matvecs;
  double tau_final;
  int64_t m_final;
  double t_reached;
  int64_t attempts;
  int32_t skipped;   /* 1: all-zero request, engine not run (integrators.py:125-127) */
  int32_t status;    /* eik_status of this call */
} EikPhipmInfo;

/* one trace row (phipm.py:341-343): attempt, t, tau, m, eps_m, omega, accepted */
typedef struct {
  int64_t attempt;
  double t;
  double tau;
  int64_t m;
  double eps_m;
  double omega;
  int64_t accepted;
} EikTraceRec;

const char* eik_last_error(void);
int eik_version(void);

/* Device cell order used by eik_swe_create (host only, no GPU needed):
 * recursive coordinate bisection of the n cell positions (px, py, pz) into
 * ntiles leaves whose sizes differ by at most one (median split along the
 * longest extent, ties by index; constant positions keep the index order).
 * ord[d] = original index of device cell d (n entries), starts[t] = first
 * device cell of leaf t (ntiles + 1 entries, starts[ntiles] = n).  Each leaf
 * is one tile of the Krylov pass.  No reference counterpart: the reference
 * has no device layout (its cell order is the grid's, swe.py:23-46). */
eik_status eik_tile_order(int64_t n, const double* px, const double* py, const double* pz,
                          int32_t ntiles, int32_t* ord, int32_t* starts);

/* ---------------------------------------------------------------- SWE */
/* ops[11] = Gx Gy Gz Dx Dy Dz Vx Vy Vz L Df (each n_g x n_g CSR).  The
 * device path applies Df as -nu * L(L .); creation returns EIK_EINVAL unless
 * the given Df equals -nu * (L @ L) entry by entry (within 1e-12 of
 * nu * sum_k |L_ik L_kj|; entries outside the pattern of L@L must be zero).
 * m_max: Krylov basis capacity (at least min(100, 4 n_g), the step path's
 * PhiTask default; eik_swe_phipm grows it for a larger task m_max, up to the
 * dense cap of 256). */
eik_status eik_swe_create(int32_t n_g, const EikCsrView* ops,
                          const double* n_x, const double* n_y,
                          const double* n_z, const double* f,
                          const double* h_s, double g, double nu,
                          int32_t device, int32_t m_max, EikSwe** out);
eik_status eik_swe_destroy(EikSwe* ctx);

/* the resident trajectory state [u_x; u_y; u_z; h] (4*n_g doubles) */
eik_status eik_swe_set_state(EikSwe* ctx, const double* u);
eik_status eik_swe_get_state(EikSwe* ctx, double* u);
/* epi3 history u_{n-1}; NULL clears it */
eik_status eik_swe_set_prev(EikSwe* ctx, const double* u_prev);

eik_status eik_swe_rhs(EikSwe* ctx, const double* u, double* out);
eik_status eik_swe_jv(EikSwe* ctx, const double* u, const double* v,
                      double* out);
eik_status eik_swe_jac_nnz(EikSwe* ctx, const double* u, int64_t* nnz);
/* same, plus the count per cell (4 rows each) into per_cell[n_g] */
eik_status eik_swe_jac_nnz_rows(EikSwe* ctx, const double* u, int64_t* nnz,
                                double* per_cell);

/* conservation diagnostics (swe.py:226-237): out = {mass, energy, potential
 * enstrophy}, each sum_i w_i q_i with w_i = weights[i] (per-cell areas) or
 * cell_area when weights is NULL.  u NULL: the resident state (no host copy).
 * EIK_EINVAL if some h <= 0. */
eik_status eik_swe_diagnostics(EikSwe* ctx, const double* u, const double* weights,
                               double cell_area, double* out);

/* phipm_simul_iom2 with A x = dt * (J(u_lin) x).  W: n x ns, column-major
 * (column i contiguous).  trace may be NULL. */
eik_status eik_swe_phipm(EikSwe* ctx, const double* u_lin, double dt,
                         const EikPhiTask* task, double* W,
                         EikPhipmInfo* info, EikTraceRec* trace,
                         int64_t trace_cap, int64_t* trace_len);

/* one step of `scheme` on the resident state (in place); calls[3] gets the
 * per-engine-call counters, *ncalls how many engine calls ran. */
eik_status eik_swe_step(EikSwe* ctx, int32_t scheme, double dt, double tol,
                        EikPhipmInfo* calls, int32_t* ncalls);
/* nsteps calls of eik_swe_step (each a CUDA-graph replay followed by one
 * host synchronisation that reads the step's status and counters back);
 * the counters are summed into matvecs/substeps; stops at the first error. */
eik_status eik_swe_advance(EikSwe* ctx, int32_t scheme, double dt, double tol,
                           int32_t nsteps, int64_t* matvecs, int64_t* substeps);

/* EngineSeeds: set != 0 stores (*tau, *m) (tau <= 0 : None), else reads */
eik_status eik_swe_seeds(EikSwe* ctx, int32_t slot, double* tau, int64_t* m,
                         int32_t set);
eik_status eik_swe_reset_seeds(EikSwe* ctx);
/* device-side snapshot of the trajectory position (state, epi3 history,
 * seeds): restore = 0 takes it, restore != 0 puts it back (stream-ordered
 * device copies, no host synchronisation).  No reference counterpart: lets a
 * caller replay the same steps (bench.py) without host traffic. */
eik_status eik_swe_snapshot(EikSwe* ctx, int32_t restore);

/* Krylov microbenchmark: reps IOM2 sweeps of dimension m (A = dt J(u)) on
 * direction v, device time of the whole launch in out[0] (ms), kept
 * dimension in out[1] */
eik_status eik_swe_krylov_bench(EikSwe* ctx, const double* u, const double* v,
                                double dt, int32_t m, int32_t reps, double* out);
/* out[9]: grid CTAs, threads/CTA, tiles, max E1, max E2, slots, compact
 * slots, compact stencil valid, dynamic smem bytes */
eik_status eik_swe_info(const EikSwe* ctx, int64_t* out);

/* EIK_PROF builds: per-phase clock64 totals of CTA 0 (16 doubles: rhs, nnz,
 * w-recurrence, Krylov, dense exp, candidate, stage perturbation, misc);
 * returns EIK_EINVAL in normal builds */
int eik_prof_read(double* out, int reset);

/* launches of libeik kernels since creation (for bench gpu_launches) */
int64_t eik_swe_launches(const EikSwe* ctx);
/* last step's per-phase device time in ms (CUDA events), engine-kernel only */
double eik_swe_last_kernel_ms(const EikSwe* ctx);
/* host-loop mode (on != 0): eik_swe_step launches the split step's kernels
 * one by one instead of replaying its CUDA graph (conditional graph nodes
 * cannot be profiled by ncu), reading the loop condition back after every
 * continuation kernel and bracketing every Krylov sweep kernel with CUDA
 * events.  Results are identical; it is slower (one host sync per sweep).
 * Also selected by the environment variable EIK_STEP_HOST at creation. */
eik_status eik_swe_set_hostloop(EikSwe* ctx, int32_t on);
/* total device time (ms, CUDA events) and number of the Krylov sweep kernels
 * run in host-loop mode since the last reset; reset != 0 zeroes them */
eik_status eik_swe_sweep_timing(EikSwe* ctx, double* ms, int64_t* nsweeps, int32_t reset);
/* Krylov iterations (IOM2 J*v) performed since creation */
int64_t eik_swe_krylov_iters(const EikSwe* ctx);
/* of those, iterations that needed the explicit orthogonalisation pass
 * (Gram-identity norm rejected for cancellation) */
int64_t eik_swe_explicit_orth(const EikSwe* ctx);

/* ---------------------------------------------------------------- CSR */
eik_status eik_csr_create(int32_t n, EikCsrView A, int32_t device,
                          int32_t m_max, EikCsr** out);
eik_status eik_csr_destroy(EikCsr* ctx);
/* A x = scale * (A_csr x); nnz_override >= 0 replaces nnz in the cost model */
eik_status eik_csr_phipm(EikCsr* ctx, double scale, int64_t nnz_override,
                         const EikPhiTask* task, double* W,
                         EikPhipmInfo* info, EikTraceRec* trace,
                         int64_t trace_cap, int64_t* trace_len);

/* ------------------------------------------------ host matvec callback */
/* The reference's MatvecOperator around an arbitrary callable
 * (phipm.py:45-54, as_operator 73-84): the engine runs on the device and
 * every matvec is one host round trip.  The callback gets x (n doubles) and
 * writes y = A x (n doubles, both host memory owned by the context), returns
 * 0 on success; any other value aborts the call with EIK_ECALLBACK.  It is
 * invoked on the thread that called eik_cb_phipm, once per performed matvec
 * (zero-skipped products are not requested), in the engine's order.
 * While the call runs, the engine's cooperative kernel holds every SM and
 * waits for the host, so the callable must be host code: a libeik entry
 * point called from inside it fails with EIK_EINVAL, eik_*_destroy calls made
 * meanwhile (finalisers, a garbage collector) are deferred until the call
 * returns, and a request left unanswered for EIK_CB_TIMEOUT_S seconds
 * (environment, default 600) -- e.g. because the callable made a call that
 * synchronises the device -- ends the call with EIK_ECALLBACK. */
typedef int (*eik_matvec_fn)(void* user, const double* x, double* y, int64_t n);
typedef struct EikCb EikCb;
eik_status eik_cb_create(int64_t n, int32_t device, int32_t m_max, EikCb** out);
eik_status eik_cb_destroy(EikCb* ctx);
/* A x = scale * callback(x); nnz is the operator's n_A for the cost model */
eik_status eik_cb_phipm(EikCb* ctx, eik_matvec_fn matvec, void* user, double scale,
                        int64_t nnz, const EikPhiTask* task, double* W,
                        EikPhipmInfo* info, EikTraceRec* trace, int64_t trace_cap,
                        int64_t* trace_len);

#ifdef __cplusplus
}
#endif

#endif /* EIK_H */
