// eik_control.h -- scalar control logic of phipm_simul_iom2, shared by the
// device engine (every CTA evaluates it redundantly on identical reduced
// inputs, so all CTAs take identical branches) and by the host unit tests.
//
// Restates /root/reference/pkg/src/expintkit/phipm.py:
//   cost_estimate      phipm.py:217-238
//   adapt_parameters   phipm.py:241-288
//   initial tau / m    phipm.py:300-313
// Python never contracts a*b+c into an FMA, so every product/sum below goes
// through eik_mul/eik_add (round-to-nearest, no contraction) to keep the
// decision arithmetic identical to CPython's.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define EIK_HD __host__ __device__ __forceinline__
#else
#define EIK_HD inline
#endif

namespace eik {

constexpr double kPadeTheta = 5.37;       // kernels.py:24
constexpr double kBreakdownTol = 1e-14;   // krylov.py:17
constexpr int kCrawlSubsteps = 100;       // phipm.py:31
constexpr int kDenseCap = 256;            // kernels.py:20

EIK_HD double eik_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
EIK_HD double eik_add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
EIK_HD double eik_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
EIK_HD double eik_div(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b;
  return r;
#endif
}

// math.ceil(x) for a finite double, as an integer
EIK_HD int64_t eik_ceil_i(double x) { return (int64_t)ceil(x); }

// phipm.py:217-238.  Returns -1 for tau <= 0 (the reference raises).
EIK_HD double cost_estimate(double tau, int64_t m, int64_t N, int64_t nA,
                            int64_t p, double norm_hhat, double t_out,
                            double t_k) {
  if (!(tau > 0.0)) return -1.0;
  double M = eik_div(44.0, 3.0);
  if (norm_hhat > kPadeTheta) {
    int64_t c = eik_ceil_i(log2(eik_div(norm_hhat, kPadeTheta)));
    M = eik_add(M, eik_mul(2.0, (double)c));
  }
  int64_t k = (t_out > t_k) ? eik_ceil_i(eik_div(eik_sub(t_out, t_k), tau)) : 1;
  int64_t pm1 = p - 1 > 0 ? p - 1 : 0;
  int64_t i12 = m * (N + nA) + 2 * pm1 * (nA + N);  // exact integer part
  int64_t d = m + p + 1;
  double f = eik_mul(M, (double)(d * d * d));
  double s = eik_add((double)i12, f);
  s = eik_add(s, (double)((2 * p + 1) * N));
  return eik_mul((double)k, s);
}

struct Adapt {
  double tau;
  int64_t m;
  int choice;  // 0 = tau, 1 = m
};

// phipm.py:241-288.  horizon = rho[-1].
EIK_HD Adapt adapt_parameters(double tau, int64_t m, double t_k, double eps,
                              double norm_hhat, double t_out, double horizon,
                              int64_t p, double tol, double delta,
                              int64_t m_max, int64_t N, int64_t nA) {
  Adapt r;
  double rem = eik_sub(horizon, t_k);
  double fl = eik_mul(tau, 1e-16);
  double remaining = rem > fl ? rem : fl;
  double omega = eik_div(eik_mul(t_out, eps), eik_mul(tau, tol));
  if (omega == 0.0) {
    double t2 = eik_mul(2.0, tau);
    r.tau = t2 < remaining ? t2 : remaining;
    r.m = m;
    r.choice = 0;
    return r;
  }
  double expo = eik_div(-1.0, (double)(p + 1));
  double tau_pred = eik_mul(tau, pow(omega, expo));
  double lo = eik_div(tau, 5.0);
  double tc = tau_pred > lo ? tau_pred : lo;
  double t2 = eik_mul(2.0, tau);
  tc = tc < t2 ? tc : t2;
  tc = tc < remaining ? tc : remaining;
  int64_t m_cap = m_max < N ? m_max : N;
  if (eik_div(remaining, tc) > (double)kCrawlSubsteps && m < m_cap) {
    r.tau = tc;
    r.m = m_cap;
    r.choice = 1;
    return r;
  }
  int64_t m_cand;
  if (omega > delta) {
    double om = omega > 1.0 ? omega : 1.0;
    m_cand = m + eik_ceil_i(log2(om));
  } else {
    m_cand = m - 1;
  }
  if (m_cand < 1) m_cand = 1;
  if (m_cand > m_cap) m_cand = m_cap;
  if (m_cand == m) {
    r.tau = tc;
    r.m = m;
    r.choice = 0;
    return r;
  }
  double tp = tau_pred > 1e-16 ? tau_pred : 1e-16;
  double nh = tau > 0.0 ? eik_div(eik_mul(norm_hhat, tau_pred), tau) : 0.0;
  double c_tau = cost_estimate(tp, m, N, nA, p, nh, t_out, t_k);
  double c_m = cost_estimate(tau, m_cand, N, nA, p, norm_hhat, t_out, t_k);
  if (c_tau <= c_m) {
    r.tau = tc;
    r.m = m;
    r.choice = 0;
  } else {
    r.tau = tau;
    r.m = m_cand;
    r.choice = 1;
  }
  return r;
}

// phipm.py:300-313: initial (tau, m).  tau_init <= 0 means "None".
EIK_HD void initial_tau_m(double tau_init, int64_t m_init, double rho0,
                          double rho_last, int64_t m_max, int64_t n,
                          double* tau, int64_t* m) {
  int64_t m_cap = m_max < n ? m_max : n;
  int64_t mm = m_init > 1 ? m_init : 1;
  *m = mm < m_cap ? mm : m_cap;
  double t = tau_init > 0.0 ? tau_init : rho0;
  double floor_ = eik_div(rho_last, 10.0 * kCrawlSubsteps);
  t = t > floor_ ? t : floor_;
  *tau = t < rho0 ? t : rho0;
}

// t ** ell / math.factorial(ell)  (phipm.py:180, 202)
EIK_HD double pow_over_fact(double t, int ell) {
  double f = 1.0;
  for (int k = 2; k <= ell; ++k) f *= (double)k;
  return eik_div(pow(t, (double)ell), f);
}

}  // namespace eik
