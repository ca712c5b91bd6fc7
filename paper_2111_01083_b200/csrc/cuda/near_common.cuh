// Shared helpers of the near-image tile kernels (near.cu, near_sym_impl.cuh).
#pragma once

#include "pw_engine.cuh"
#include "pw_math.cuh"

namespace pwb {

// Fused layouts (every near image, cell.cpp:47-58) have shift.y = n*eta = 0 on the
// middle row and shift = (0, 0) at its centre; (dy) - 0.0 == dy exactly, so those
// subtractions are skipped at compile time. A single-image launch (1x1) knows nothing.
template <int NXI, int NROW>
__device__ __forceinline__ double row_dy(double dy, const NearArgs& a, int n) {
  constexpr bool fused = !(NXI == 1 && NROW == 1);
  if (fused && n == NROW / 2) return dy;
  return dy - a.shy[n];
}
// USK (unskewed cell, xi == 0): shx[n][m] = m d + n * 0.0 = m d for every row n, so every
// row reads the middle row's shift -- the same value -- and the compiler forms each column's
// rx once per pair instead of once per image (bitwise the same numbers).
template <int NXI, int NROW, bool USK = false>
__device__ __forceinline__ double img_dx(double dx, const NearArgs& a, int n, int m) {
  constexpr bool fused = !(NXI == 1 && NROW == 1);
  if (USK) n = NROW / 2;
  if (fused && n == NROW / 2 && m == NXI / 2) return dx;
  return dx - a.shx[n * NXI + m];
}

// Range [X_lo, X_hi] of X = beta^2 |(t - s) - shift|^2 over t in the target box and s in
// the source box; boxes are (xmin, -xmax, ymin, -ymax). Used for the screened tiles'
// image masks and per-tile-pair regimes (pw_math.cuh regime_of).
__device__ __forceinline__ void image_xrange(const double* tb, const double* sb, double shx, double shy,
                                             double beta2, double& X_lo, double& X_hi) {
  const double xlo = (tb[0] + sb[1]) - shx;  // txmin - sxmax - shift
  const double xhi = (-tb[1] - sb[0]) - shx;
  const double ylo = (tb[2] + sb[3]) - shy;
  const double yhi = (-tb[3] - sb[2]) - shy;
  const double gx = xlo > 0.0 ? xlo : (xhi < 0.0 ? -xhi : 0.0);
  const double gy = ylo > 0.0 ? ylo : (yhi < 0.0 ? -yhi : 0.0);
  const double mx = fmax(fabs(xlo), fabs(xhi)), my = fmax(fabs(ylo), fabs(yhi));
  X_lo = beta2 * fma(gx, gx, gy * gy);
  X_hi = beta2 * fma(mx, mx, my * my);
}

// Axis-aligned box (xmin, -xmax, ymin, -ymax) of a point set, warp-reduced; lane 0 of
// each warp stores its warp's box in s_box (4 doubles).
__device__ __forceinline__ void warp_box_store(double b0, double b1, double b2, double b3, int lane, double* s_box) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    b0 = fmin(b0, __shfl_xor_sync(0xffffffffu, b0, o));
    b1 = fmin(b1, __shfl_xor_sync(0xffffffffu, b1, o));
    b2 = fmin(b2, __shfl_xor_sync(0xffffffffu, b2, o));
    b3 = fmin(b3, __shfl_xor_sync(0xffffffffu, b3, o));
  }
  if (lane == 0) {
    s_box[0] = b0;
    s_box[1] = b1;
    s_box[2] = b2;
    s_box[3] = b3;
  }
}

}  // namespace pwb
