// Host build of csrc/eik_control.h (the device controller's logic) for the
// CPU unit tests: the very same source the engine kernel evaluates.
#include "../../paper_1805_02144_b200/csrc/eik_control.h"

extern "C" {
double t_cost(double tau, long long m, long long N, long long nA, long long p,
              double nh, double t_out, double t_k) {
  return eik::cost_estimate(tau, m, N, nA, p, nh, t_out, t_k);
}
void t_adapt(double tau, long long m, double t_k, double eps, double nh,
             double t_out, double horizon, long long p, double tol, double delta,
             long long m_max, long long N, long long nA, double* tau_out,
             long long* m_out) {
  eik::Adapt a = eik::adapt_parameters(tau, m, t_k, eps, nh, t_out, horizon, p, tol,
                                       delta, m_max, N, nA);
  *tau_out = a.tau;
  *m_out = a.m;
}
void t_init(double tau_init, long long m_init, double rho0, double rho_last,
            long long m_max, long long n, double* tau, long long* m) {
  int64_t mm;
  eik::initial_tau_m(tau_init, m_init, rho0, rho_last, m_max, n, tau, &mm);
  *m = mm;
}
double t_powfact(double t, int ell) { return eik::pow_over_fact(t, ell); }
}
