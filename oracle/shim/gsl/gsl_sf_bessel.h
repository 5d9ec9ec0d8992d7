// ORACLE TEST INFRASTRUCTURE — not product code.
//
// From-scratch stand-in for the one GSL entry point the reference kernel TU
// calls (proj/core/src/kernel.cpp:42, general-nu Matern only; no BASELINE
// config reaches it). GSL is not installed in this image.
// log K_nu(x) is computed from the C++17 special function; where K_nu
// overflows, the small-x leading term log(Gamma(nu)/2) + nu log(2/x) is used.
#pragma once

#include <cmath>
#include <limits>

typedef struct {
  double val;
  double err;
} gsl_sf_result;

static inline int gsl_sf_bessel_lnKnu_e(const double nu, const double x,
                                        gsl_sf_result* result) {
  if (!(x > 0.0) || nu < 0.0) {
    result->val = std::numeric_limits<double>::quiet_NaN();
    result->err = std::numeric_limits<double>::quiet_NaN();
    return 1;  // GSL_EDOM
  }
  double k = std::cyl_bessel_k(nu, x);
  double v;
  if (std::isfinite(k) && k > 0.0) {
    v = std::log(k);
  } else if (!std::isfinite(k)) {
    v = std::lgamma(nu) - std::log(2.0) + nu * std::log(2.0 / x);
  } else {  // underflow at very large x: K_nu(x) ~ sqrt(pi/(2x)) e^{-x}
    v = 0.5 * std::log(M_PI / (2.0 * x)) - x;
  }
  result->val = v;
  result->err = 2.0 * std::numeric_limits<double>::epsilon() * std::fabs(v);
  return 0;
}
