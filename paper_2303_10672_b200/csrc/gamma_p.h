/* Regularized lower incomplete gamma P(a, x).
 *
 * Stand-in for boost::math::gamma_p, the one third-party arithmetic routine
 * on the table-building path (reference: proj/src/dist.cpp:3,15-18; Boost
 * version unpinned, proj/CMakeLists.txt:16). Boost is not in this image, so
 * both the engine's table builder and the oracle build of the reference use
 * this one definition; the demand pmf they feed the kernels is therefore
 * bit-identical by construction. Accuracy is pinned against the 50-digit
 * frozen values of proj/tests/test_dist.cpp:43-49 (1e-10) in tests/.
 *
 * Algorithm: power series for x < a + 1, modified-Lentz continued fraction
 * for the complement Q otherwise (the classical split; both converge to
 * < 1e-17 relative).  Plain C so the C oracle can include it too.
 */
#ifndef PVI_B200_GAMMA_P_H
#define PVI_B200_GAMMA_P_H

#include <math.h>

static inline double pvi_gamma_p(double a, double x) {
  if (x <= 0.0) return 0.0;
  const double log_prefactor = -x + a * log(x) - lgamma(a);
  if (x < a + 1.0) {
    double denom = a;
    double term = 1.0 / a;
    double sum = term;
    for (int n = 0; n < 100000; ++n) {
      denom += 1.0;
      term *= x / denom;
      sum += term;
      if (fabs(term) < fabs(sum) * 1e-17) break;
    }
    return sum * exp(log_prefactor);
  }
  const double tiny = 1e-300;
  double b = x + 1.0 - a;
  double c = 1.0 / tiny;
  double d = 1.0 / b;
  double h = d;
  for (int i = 1; i < 100000; ++i) {
    const double an = -i * (i - a);
    b += 2.0;
    d = an * d + b;
    if (fabs(d) < tiny) d = tiny;
    c = b + an / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double delta = d * c;
    h *= delta;
    if (fabs(delta - 1.0) < 1e-17) break;
  }
  return 1.0 - exp(log_prefactor) * h;
}

#endif
