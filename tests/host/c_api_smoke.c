/* Plain-C client of libeik.so (include/eik.h): builds a tiny operator set
 * (a 16x16 doubly periodic plane, the reference's planar factory layout),
 * runs F(u), J v, two EXPRB4 steps and the diagnostics, and checks basic
 * invariants.  Compiled and run by tests/test_gpu_c_api.py on the GPU box. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "eik.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define NX 16
#define N (NX * NX)

typedef struct { int32_t indptr[N + 1]; int32_t idx[N * 5]; double val[N * 5]; int64_t nnz; } Csr;

static int id(int x, int y) { return ((y + NX) % NX) * NX + (x + NX) % NX; }

static void build(Csr* m, double cx, double cy, double c0, double cl) {
  /* row i: c0*u_i + cx*(u_e - u_w) + cy*(u_n - u_s) + cl*(sum of 4 nbrs) */
  int64_t k = 0;
  for (int y = 0; y < NX; ++y)
    for (int x = 0; x < NX; ++x) {
      int i = id(x, y);
      m->indptr[i] = (int32_t)k;
      int cols[5] = {id(x, y - 1), id(x - 1, y), i, id(x + 1, y), id(x, y + 1)};
      double v[5] = {-cy + cl, -cx + cl, c0, cx + cl, cy + cl};
      /* sort columns ascending (CSR canonical) */
      for (int a = 0; a < 5; ++a)
        for (int b = a + 1; b < 5; ++b)
          if (cols[b] < cols[a]) { int t = cols[a]; cols[a] = cols[b]; cols[b] = t;
                                   double tv = v[a]; v[a] = v[b]; v[b] = tv; }
      for (int a = 0; a < 5; ++a) { m->idx[k] = cols[a]; m->val[k] = v[a]; ++k; }
    }
  m->indptr[N] = (int32_t)k;
  m->nnz = k;
}

int main(void) {
  const double dx = 1.0e5, g = 9.80616, f0 = 1e-4;
  static Csr ddx, ddy, zero, vx, vy, lap;
  build(&ddx, 1.0 / (2 * dx), 0, 0, 0);
  build(&ddy, 0, 1.0 / (2 * dx), 0, 0);
  build(&vx, 0, -1.0 / (2 * dx), 0, 0);
  build(&vy, 1.0 / (2 * dx), 0, 0, 0);
  build(&lap, 0, 0, -4.0 / (dx * dx), 1.0 / (dx * dx));
  memset(&zero, 0, sizeof(zero));
  const double nu = 0.04e-2 * pow(dx, 4) / 240.0;
  /* Df = -nu * lap @ lap (13-point), dense accumulation per row */
  int32_t* dfp = malloc((N + 1) * sizeof(int32_t));
  int32_t* dfi = malloc(N * 13 * sizeof(int32_t));
  double* dfv = malloc(N * 13 * sizeof(double));
  int64_t k = 0;
  for (int i = 0; i < N; ++i) {
    double row[N];
    memset(row, 0, sizeof(row));
    for (int a = lap.indptr[i]; a < lap.indptr[i + 1]; ++a) {
      int j = lap.idx[a];
      for (int b = lap.indptr[j]; b < lap.indptr[j + 1]; ++b) row[lap.idx[b]] += lap.val[a] * lap.val[b];
    }
    dfp[i] = (int32_t)k;
    for (int j = 0; j < N; ++j) if (row[j] != 0.0) { dfi[k] = j; dfv[k] = -nu * row[j]; ++k; }
  }
  dfp[N] = (int32_t)k;
  EikCsrView zv = {0, zero.indptr, zero.idx, zero.val};
  EikCsrView ops[11] = {
      {ddx.nnz, ddx.indptr, ddx.idx, ddx.val}, {ddy.nnz, ddy.indptr, ddy.idx, ddy.val}, zv,
      {ddx.nnz, ddx.indptr, ddx.idx, ddx.val}, {ddy.nnz, ddy.indptr, ddy.idx, ddy.val}, zv,
      {vx.nnz, vx.indptr, vx.idx, vx.val},     {vy.nnz, vy.indptr, vy.idx, vy.val},     zv,
      {lap.nnz, lap.indptr, lap.idx, lap.val}, {k, dfp, dfi, dfv}};
  static double nxa[N], nya[N], nza[N], fa[N], hs[N], u[4 * N], out[4 * N], v[4 * N];
  for (int i = 0; i < N; ++i) { nza[i] = 1.0; fa[i] = f0; }
  for (int i = 0; i < N; ++i) {
    int x = i % NX, y = i / NX;
    u[i] = 5.0 * sin(2 * M_PI * y / NX);
    u[N + i] = 5.0 * sin(2 * M_PI * x / NX);
    u[3 * N + i] = 8000.0 + 50.0 * cos(2 * M_PI * x / NX) * cos(2 * M_PI * y / NX);
    v[i] = 1.0; v[3 * N + i] = (double)(i % 7);
  }
  EikSwe* ctx = NULL;
  if (eik_swe_create(N, ops, nxa, nya, nza, fa, hs, g, nu, 0, 100, &ctx) != EIK_OK) {
    printf("create failed: %s\n", eik_last_error()); return 1;
  }
  if (eik_swe_rhs(ctx, u, out) != EIK_OK) { printf("rhs: %s\n", eik_last_error()); return 1; }
  double s = 0; for (int i = 0; i < 4 * N; ++i) s += fabs(out[i]);
  int64_t nnz = 0;
  if (eik_swe_jv(ctx, u, v, out) != EIK_OK || eik_swe_jac_nnz(ctx, u, &nnz) != EIK_OK) {
    printf("jv/nnz: %s\n", eik_last_error()); return 1;
  }
  double d0[3], d1[3];
  eik_swe_set_state(ctx, u);
  eik_swe_diagnostics(ctx, NULL, NULL, dx * dx, d0);
  for (int step = 0; step < 2; ++step) {
    EikPhipmInfo calls[3]; int32_t nc = 0;
    if (eik_swe_step(ctx, EIK_EXPRB42, 600.0, 1e-8, calls, &nc) != EIK_OK) {
      printf("step: %s\n", eik_last_error()); return 1;
    }
    printf("step %d: calls %d, matvecs %lld/%lld, m %lld/%lld\n", step, nc,
           (long long)calls[0].matvecs, (long long)calls[1].matvecs,
           (long long)calls[0].m_final, (long long)calls[1].m_final);
  }
  eik_swe_diagnostics(ctx, NULL, NULL, dx * dx, d1);
  double drift = fabs(d1[0] - d0[0]) / d0[0];
  printf("rhs |F|_1 %.6e, nnz(J) %lld, mass drift %.3e\n", s, (long long)nnz, drift);
  eik_swe_destroy(ctx);
  free(dfp); free(dfi); free(dfv);
  if (!(s > 0) || nnz <= 0 || drift > 1e-12) return 2;
  printf("C ABI OK\n");
  return 0;
}
