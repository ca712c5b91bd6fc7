// TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
//
// Stand-in for the GSL special functions the reference links
// (/root/reference/proj/src/kernels.cpp:13-21, :78-96). GSL is absent from the
// image and unpinned by the reference (/root/reference/proj/CMakeLists.txt:12);
// its published contract is e^x K_n(x) for x > 0 and a domain error otherwise.
// Pinned by the reference's own known answers (proj/tests/test_kernels.cpp:28-48)
// in tests/test_oracle_pins.py.
//
// Two modes (env ORACLE_BESSEL):
//   accurate : std::cyl_bessel_k (libstdc++), ~1 ulp but ~400 ns per call;
//   fast     : ascending series for x <= 2, and for x > 2 the trapezoidal rule on
//              e^x K_n(x) = int_0^inf exp(-x (cosh t - 1)) cosh(n t) dt, which
//              converges geometrically in the step (the integrand is entire and
//              bounded on the strip |Im t| < pi/2).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "gsl/gsl_errno.h"
#include "gsl/gsl_sf_bessel.h"

namespace {

constexpr double kEulerGamma = 0.57721566490153286060651209008240243;

bool accurate_mode() {
  static const bool acc = [] {
    const char* v = std::getenv("ORACLE_BESSEL");
    return v && std::strcmp(v, "accurate") == 0;
  }();
  return acc;
}

// Ascending series (Abramowitz & Stegun 9.6.13 and 9.6.11 with n = 1), x <= 2.
void series_k01(double x, double* k0, double* k1) {
  const double t = 0.25 * x * x;
  const double lhalf = std::log(0.5 * x);
  double i0 = 0.0, s0 = 0.0;    // sum t^k/(k!)^2 and sum H_k t^k/(k!)^2
  double i1 = 0.0, s1 = 0.0;    // sum t^k/(k!(k+1)!) and its digamma-weighted companion
  double term0 = 1.0;           // t^k/(k!)^2
  double term1 = 1.0;           // t^k/(k!(k+1)!)
  double hk = 0.0;              // harmonic number H_k
  for (int k = 0; k < 40; ++k) {
    i0 += term0;
    s0 += hk * term0;
    i1 += term1;
    const double hk1 = hk + 1.0 / (k + 1.0);
    // psi(k+1) + psi(k+2) = H_k + H_{k+1} - 2 gamma
    s1 += (hk + hk1 - 2.0 * kEulerGamma) * term1;
    term0 *= t / ((k + 1.0) * (k + 1.0));
    term1 *= t / ((k + 1.0) * (k + 2.0));
    hk = hk1;
    if (term0 < 1e-19 * i0 && term1 < 1e-19 * i1) break;
  }
  *k0 = -(lhalf + kEulerGamma) * i0 + s0;
  const double I1 = 0.5 * x * i1;
  *k1 = 1.0 / x + lhalf * I1 - 0.25 * x * s1;
}

// Step shrinks like 1/sqrt(x): the integrand is a Gaussian of width ~1/sqrt(x) and
// the strip of analyticity that controls the error narrows the same way.
// x (cosh t - 1) = 2 x sinh^2(t/2) avoids the cancellation at small t.
double trapezoid_scaled(int n, double x) {
  const double h = std::min(0.125, 0.5 / std::sqrt(x));
  double acc = 0.5;  // t = 0 contributes 1/2 * exp(0) * cosh(0)
  for (int k = 1; k < 100000; ++k) {
    const double t = k * h;
    const double sh = std::sinh(0.5 * t);
    const double a = 2.0 * x * sh * sh;
    const double e = a - n * t;
    acc += (n == 0) ? std::exp(-a) : std::exp(-a) * std::cosh(n * t);
    if (e > 45.0) break;
  }
  return h * acc;
}

double fast_scaled(int n, double x) {
  if (x <= 2.0) {
    double k0, k1;
    series_k01(x, &k0, &k1);
    const double ex = std::exp(x);
    if (n == 0) return k0 * ex;
    if (n == 1) return k1 * ex;
    double km = k0 * ex, kc = k1 * ex;
    for (int l = 1; l < n; ++l) {
      const double kn = km + (2.0 * l / x) * kc;
      km = kc;
      kc = kn;
    }
    return kc;
  }
  if (n <= 1) return trapezoid_scaled(n, x);
  double km = trapezoid_scaled(0, x), kc = trapezoid_scaled(1, x);
  for (int l = 1; l < n; ++l) {
    const double kn = km + (2.0 * l / x) * kc;
    km = kc;
    kc = kn;
  }
  return kc;
}

double accurate_scaled(int n, double x) {
  if (x > 600.0) return fast_scaled(n, x);  // cyl_bessel_k underflows; the scaled value does not
  return std::cyl_bessel_k(static_cast<double>(n), x) * std::exp(x);
}

int eval(int n, double x, gsl_sf_result* r) {
  if (!(x > 0.0) || n < 0) {
    r->val = NAN;
    r->err = NAN;
    return GSL_EDOM;
  }
  r->val = accurate_mode() ? accurate_scaled(n, x) : fast_scaled(n, x);
  r->err = 4e-16 * std::fabs(r->val);
  return GSL_SUCCESS;
}

}  // namespace

extern "C" {

gsl_error_handler_t* gsl_set_error_handler_off(void) { return nullptr; }

const char* gsl_strerror(int gsl_errno) {
  switch (gsl_errno) {
    case GSL_SUCCESS: return "success";
    case GSL_EDOM: return "input domain error";
    case GSL_EUNDRFLW: return "underflow";
    default: return "unknown error";
  }
}

int gsl_sf_bessel_K0_scaled_e(double x, gsl_sf_result* r) { return eval(0, x, r); }
int gsl_sf_bessel_K1_scaled_e(double x, gsl_sf_result* r) { return eval(1, x, r); }
int gsl_sf_bessel_Kn_scaled_e(int n, double x, gsl_sf_result* r) { return eval(n, x, r); }

}  // extern "C"
