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
template <int NXI, int NROW>
__device__ __forceinline__ double img_dx(double dx, const NearArgs& a, int n, int m) {
  constexpr bool fused = !(NXI == 1 && NROW == 1);
  if (fused && n == NROW / 2 && m == NXI / 2) return dx;
  return dx - a.shx[n * NXI + m];
}

}  // namespace pwb
