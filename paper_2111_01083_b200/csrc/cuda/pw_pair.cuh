// Per-pair kernel math shared by the device P2P tiles and the host API.
// Restates /root/reference/proj/src/kernels.cpp:36-68 (ModStokes g1/g2) with the
// series coefficients of pw_coeffs.h.
#pragma once

#include "pw_math.cuh"

namespace pwk {

struct G12 {
  double g1, g2;
};

// g1(z) = 1 - z K1(z), g2(z) = -1 + z K1(z) + z^2 K0(z) (kernels.cpp:32-68).
// For z < 0.5 both are O(z^2 log z) and the direct form cancels, so the
// ascending series is used: with q = z^2/4, lh = ln(z/2),
//   g1 = q (B1S(q) - 2 lh I1S(q)),  K0 = -(lh + gamma) I0S(q) + A0S(q).
PW_HD G12 mod_stokes_g12(double z) {
  G12 o;
  const double X = z * z;
  if (z >= 0.5) {
    const K01 k = k01_of_sq(X);
    const double zk1 = k.k1_over_x * X;
    o.g1 = 1.0 - zk1;
    o.g2 = -o.g1 + X * k.k0;
    return o;
  }
  const double q = 0.25 * X;
  const double lh = 0.5 * log_pos(q);
  const double k0 = fma(-(lh + PW_EULER_GAMMA), pw_poly_i0s(q), pw_poly_a0s(q));
  o.g1 = q * fma(-2.0 * lh, pw_poly_i1s(q), pw_poly_b1s(q));
  o.g2 = -o.g1 + X * k0;
  return o;
}

// ln(rx^2 + ry^2) for any finite nonzero (rx, ry), including squares that
// underflow (rare slow path of the fused tiles).
PW_HD double log_r2_safe(double rx, double ry) {
  double ax = fabs(rx), ay = fabs(ry);
  double big = ax > ay ? ax : ay;
  if (big > 1e-150 && big < 1e150) return log_pos(fma(rx, rx, ry * ry));
  const double scale = big <= 1e-150 ? 0x1p600 : 0x1p-600;
  const double sx = rx * scale, sy = ry * scale;
  const double shift = big <= 1e-150 ? -1200.0 : 1200.0;
  return fma(shift, kLn2Hi, fma(shift, kLn2Lo, log_pos(fma(sx, sx, sy * sy))));
}

}  // namespace pwk
