/* The tiled pass's division by a shared reciprocal (csrc/eik_dev.cuh, form_x)
 * against IEEE division: r = 1/h, q0 = a r, q = fma(fma(-q0, h, a), r, q0).
 * Prints the number of mismatches over n random pairs (argv[1]) with
 * exponents like the Krylov vectors' (|a| in 2^-60..2^20, h in 2^-40..2^40). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double mk(int emin, int emax) {
  uint64_t m = rnd() & 0xFFFFFFFFFFFFFULL;
  int e = emin + (int)(rnd() % (uint64_t)(emax - emin + 1));
  uint64_t b = ((uint64_t)(e + 1023) << 52) | m | ((rnd() & 1) << 63);
  double d;
  memcpy(&d, &b, 8);
  return d;
}
static double shdiv(double a, double h) {
  const double r = 1.0 / h, q0 = a * r;
  return fma(fma(-q0, h, a), r, q0);
}
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 20000000L, bad = 0;
  for (long i = 0; i < n; ++i) {
    const double a = mk(-60, 20), h = fabs(mk(-40, 40));
    if (shdiv(a, h) != a / h) ++bad;
  }
  /* exact cases */
  if (shdiv(0.0, 3.0) != 0.0 || shdiv(6.0, 3.0) != 2.0 || shdiv(-1.0, 4.0) != -0.25) ++bad;
  printf("%ld\n", bad);
  return 0;
}
