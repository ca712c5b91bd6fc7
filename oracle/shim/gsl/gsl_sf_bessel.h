/* TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
 *
 * GSL-shaped scaled modified Bessel K_n used by the reference
 * (/root/reference/proj/src/kernels.cpp:78-96). The values are e^x K_n(x).
 * Implementation: oracle/shim/bessel_shim.cpp. Two evaluation modes,
 * selected by the environment variable ORACLE_BESSEL:
 *   "accurate" -> libstdc++ std::cyl_bessel_k (about 1 ulp, slow);
 *   anything else (default "fast") -> own ascending series (x <= 2) and a
 *     trapezoidal rule on the integral K_n(x) = int_0^inf e^{-x cosh t}
 *     cosh(n t) dt (x > 2), agreeing with "accurate" to <= 2e-15 relative
 *     (tests/test_oracle_pins.py).
 */
#ifndef ORACLE_SHIM_GSL_SF_BESSEL_H
#define ORACLE_SHIM_GSL_SF_BESSEL_H

#include "gsl_errno.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double val;
  double err;
} gsl_sf_result;

int gsl_sf_bessel_K0_scaled_e(double x, gsl_sf_result* result);
int gsl_sf_bessel_K1_scaled_e(double x, gsl_sf_result* result);
int gsl_sf_bessel_Kn_scaled_e(int n, double x, gsl_sf_result* result);

#ifdef __cplusplus
}
#endif

#endif
