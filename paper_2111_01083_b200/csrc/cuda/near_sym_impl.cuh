// Symmetric near-image P2P for targets == sources (configs c1, c3, c4, c5).
//
// The near image set is symmetric (shift <-> -shift, cell.cpp:47-58), so the
// image-summed kernel of a pair satisfies G3(t_l - s_j) = +/- G3(t_j - s_l)
// (even part: log, K0, Stokeslet tensor; odd part: gradient, pressurelet). Each
// unordered pair is evaluated once and feeds both its row (target l, weight w_j)
// and its column (target j, weight w_l): half the transcendental work of the
// one-sided tile (near.cu). Exact-zero semantics are unchanged: an exact zero of
// (t_l - s_j) - shift is an exact zero of (t_j - s_l) + shift (negation is exact),
// identity-image self pairs are skipped, any other coincidence sets the flag.
//
// Work items: row tile I (TILE = 128 * TPT points, TPT per thread) x a chunk of
// column tiles (CT = 128 * CPT points, CT dividing TILE) starting at the row tile's
// own first column tile; the column tiles inside the row tile run one-sided (each
// ordered pair once, self pairs included), the ones beyond it symmetric. Column
// partials use a rotating schedule (lane l reads column (l + i) mod CT, one private
// column copy per warp) so no two lanes of a warp touch the same column and no
// atomics are needed inside the block.
//
// Screened kernels (modified Helmholtz): off-diagonal tile pairs run image-outer
// sweeps with a per-tile-pair image mask and regime (bounding boxes of both tiles),
// see the CULL functor and DESIGN.md §3.1 items 8-10.
//
// Fast path: for kernels whose per-pair work is a product of image distances
// (Laplace log, Stokeslet) the off-diagonal tiles run branch-free; a pair whose
// product is 0 / subnormal / inf (exact coincidence, extreme scales) only raises
// a flag, and a tile that saw one is redone on the careful per-image path.
//
// Row and column sums leave the block through integer atomics on a 3-limb
// fixed-point accumulator (resolution 2^-62, range 2^64): integer addition is
// associative, so the result is bitwise deterministic for any schedule, and it
// is converted back to fp64 once at the end.
//
// This header holds the templates (functors, the tile kernel, its launcher); the
// explicit instantiations are split per kernel family across near_sym_laplace.cu,
// near_sym_modhelm.cu and near_sym_stokes.cu so they compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "near_common.cuh"
#include "pw_engine.cuh"
#include "pw_math.cuh"
#include "pw_pair.cuh"

namespace pwb {
namespace sym {


#ifndef PWB_SYM_LAPLACE_TPT
#define PWB_SYM_LAPLACE_TPT 4  // targets per thread of the Laplace tile
#endif
#ifndef PWB_SYM_MH_UNROLL_M
#define PWB_SYM_MH_UNROLL_M 3  // image columns per unrolled step of the screened symmetric tile (c5 slice: 1 -> 573 ms, 3 -> 480)
#endif
#ifndef PWB_SYM_MH_SRC_UNROLL
#define PWB_SYM_MH_SRC_UNROLL 8  // sources per unrolled step of the screened image-outer sweeps (c5 slice: 2 -> 159 ms, 4 -> 154; c5 full, r3x: 2 -> 138.9 s, 4 -> 132.1, 6 -> 127.9, 8 -> 127.1)
#endif
#ifndef PWB_SYM_MH_GEN_UNROLL
#define PWB_SYM_MH_GEN_UNROLL 1  // sources per unrolled step of the per-pair-dispatch sweep (c5 slice: 4 -> 153.6 ms, 1 -> 143.7)
#endif
#ifndef PWB_SYM_MH_NEAR_SWEEP
#define PWB_SYM_MH_NEAR_SWEEP 1  // 1: a tile pair wholly in 2 <= x < 6 gets its own branch-free sweep (c5: 143.7 vs 153.0 without)
#endif
#ifndef PWB_SYM_MH_TPT
#define PWB_SYM_MH_TPT 2  // targets per thread of the screened symmetric tile
#endif
#ifndef PWB_SYM_LAPLACE_UNROLL
#define PWB_SYM_LAPLACE_UNROLL 4  // sources per unrolled step of the fast loop (c4: 904 -> 895 ms vs 2)
#endif
#ifndef PWB_SYM_LOG_TABLE
#define PWB_SYM_LOG_TABLE 1  // reduced tier: table-driven ln (pw_math.cuh log_tab) instead of log_pos_k<true>
#endif
#ifndef PWB_SYM_LAPLACE_CPT
#define PWB_SYM_LAPLACE_CPT 1  // column points per thread of the Laplace tile (column tile 128 * CPT; c4: 4 -> 669 ms, 2 -> 667, 1 at 7 blocks -> 653)
#endif
#ifndef PWB_SYM_LAPLACE_REPL
#define PWB_SYM_LAPLACE_REPL 8  // log-table replicas of the Laplace tile (8: conflict-free LDS.128)
#endif
#ifndef PWB_SYM_CLOG_REPL
#define PWB_SYM_CLOG_REPL 4  // replicas of the coarse (256-entry) table: 4 x 4 KB keeps 7 blocks/SM
#endif
#ifndef PWB_SYM_CLOG_TAB
#define PWB_SYM_CLOG_TAB 8  // coarse table code (pw_math.cuh tab_bits / log_f_deg): 8 = 256 x degree 2
#endif
#ifndef PWB_SYM_STOKES_TPT
#define PWB_SYM_STOKES_TPT 2  // targets per thread of the Stokeslet tile
#endif
#ifndef PWB_SYM_STOKES_CPT
#define PWB_SYM_STOKES_CPT 2  // column points per thread of the Stokeslet tile
#endif
#ifndef PWB_SYM_STOKES_UNROLL
#define PWB_SYM_STOKES_UNROLL 2  // sources per unrolled step of the Stokeslet tile's fast loop
#endif
#ifndef PWB_SYM_STOKES_MINB
#define PWB_SYM_STOKES_MINB 0  // 0: ptxas's own register allocation (166 registers, 3 blocks/SM)
#endif
#ifndef PWB_SYM_KEEP_SMEM
#define PWB_SYM_KEEP_SMEM 0  // 1: the fast path's pre-tile row sums live in shared memory (frees registers)
#endif
#ifndef PWB_SYM_LAPLACE_MINB
#define PWB_SYM_LAPLACE_MINB 8  // 8 x 4 warps/SM at 64 registers (the cold careful path spills 32 B): c4 near 637.3 / 639.1 -> 632.9 / 632.7 ms vs 7 (r2i, r2j); 7 beat 6 (667 -> 653)
#endif
// Shape of the product-form Laplace tile (SymLaplace PROD). Fewer, fatter threads than the
// image-loop tile: with 14.25 fp64 per pair the per-source work (three LDS, the column
// partial's read-modify-write, index arithmetic) and the dependent chains weigh more, and 8
// targets per thread at 4 blocks/SM (128 registers) beat 4 targets at 8 blocks (A/B r3c/r3d,
// c4 near: TPT 4 / 8 blocks / unroll 4: 571 ms; TPT 6 / 5 blocks / unroll 2: 552;
// TPT 8 / 4 blocks: unroll 1 549, unroll 2 542, unroll 4 560; + 256-point column tiles 539;
// TPT 10 / 3 blocks 547; TPT 12 / 3 blocks 552; TPT 16 / 2 blocks 576).
#ifndef PWB_SYM_PROD_TPT
#define PWB_SYM_PROD_TPT 8
#endif
#ifndef PWB_SYM_PROD_CPT
#define PWB_SYM_PROD_CPT 2  // column tile 256 points
#endif
#ifndef PWB_SYM_PROD_MINB
#define PWB_SYM_PROD_MINB 4
#endif
#ifndef PWB_SYM_PROD_UNROLL
#define PWB_SYM_PROD_UNROLL 2
#endif
#ifndef PWB_SYM_PROD_ITEM_SOURCES
#define PWB_SYM_PROD_ITEM_SOURCES 1024  // sources per work item: 0.66 ms items, so an 8-rank split's last wave costs ~1 % (4096: 2.7 ms items, 8-rank near efficiency 0.93, r3p)
#endif
#ifndef PWB_SYM_PROD_THREADS
#define PWB_SYM_PROD_THREADS 128  // threads per block (A/B r2w: 256 with one 8-replica table per 8 warps 608 ms vs 572)
#endif
#ifndef PWB_SYM_PROD_REPL
#define PWB_SYM_PROD_REPL 8  // log-table replicas: 8 = conflict-free LDS.128 (32 KB at 256 entries, fits 4 blocks/SM; 4: 545 vs 542 ms)
#endif
#ifndef PWB_SYM_PROD_SEED
#define PWB_SYM_PROD_SEED 0  // 1: reciprocal-seeded 8-byte table (pw_math.cuh log_seed): half the table bytes, +2.8 instructions per pair; A/B r2w 599 ms vs 572
#endif
// Threads per block: K::THREADS (128 unless a functor says otherwise); a row tile is
// K::THREADS * K::TPT points, a column tile kColUnit * K::CPT points.
constexpr int kColUnit = 128;
constexpr int kSymMhUnrollM = PWB_SYM_MH_UNROLL_M;
constexpr int kSymMhSrcUnroll = PWB_SYM_MH_SRC_UNROLL;

// ---------------------------------------------------------------- fixed point
// v = a 2^22 + b 2^-20 + c 2^-62; limbs truncate toward zero so each carries the
// sign of v and each remainder is exact. Layout: target-major, the three limbs of
// output c of target l at acc[(l * nout + c) * 3 + {0,1,2}], so a contiguous slice of
// targets is a contiguous slice of the buffer (the multi-GPU reduce-scatter operand).
//
// Values are scaled by an exact power of two 2^k before the split (and by 2^-k in the
// readout), k = fx_exponent(max |strength|, n): the scaled sum over all n sources of
// |strength| stays below 2^24, so the accumulator's resolution and range follow the
// strengths the way fp64 summation does (the reference sums in plain fp64,
// apply.cpp:532-540) -- strengths of 1e-15 or 1e15 give the same relative accuracy as
// O(1) ones. A scaled value at or beyond 2^84 (limb a would overflow), inf or NaN raises
// flag bit 1 (value 2) and the engine redoes the near field on the one-sided fp64 tile
// (engine.cu Plan::near). The scale is re-read at each flush (one cached load per
// thread and column tile) rather than held in a register across the tile loop.
__device__ __forceinline__ void fx_add(unsigned long long* p, double v, const NearArgs& na) {
  v *= fx_scale(fx_exponent(*na.fx_maxhi, na.ns));
  if (!(fabs(v) < 0x1p84)) {
    atomicOr(na.flag, 2);
    return;
  }
  const double a = trunc(v * 0x1p-22);
  const double r1 = fma(-a, 0x1p22, v);
  const double b = trunc(r1 * 0x1p20);
  const double r2 = fma(-b, 0x1p-20, r1);
  const double c = rint(r2 * 0x1p62);
  atomicAdd(p, static_cast<unsigned long long>(static_cast<long long>(a)));
  atomicAdd(p + 1, static_cast<unsigned long long>(static_cast<long long>(b)));
  atomicAdd(p + 2, static_cast<unsigned long long>(static_cast<long long>(c)));
}

// ---------------------------------------------------------------- symmetric pair values
// NV image-summed values per pair; row(acc, V, w_j) and col(acc, V, w_l) contract
// them with the other side's strength (col flips the odd components).
// values():      careful per-image semantics (slow path included, sets `flag`);
// values_fast(): branch-free, only valid when `bad` stays 0 (FAST kernels).

// PROD (one image row of three, binned points pre-scaled by a.prod_sc = 2 / d so the period
// is 2): the three images' product in closed form. With u = dx^2, w = u + dy^2,
//   r0^2 r-^2 r+^2 = w ((w + d^2)^2 - 4 d^2 u);
// in the tile's units U = dX^2, W = U + dY^2, a = W / 4 + 1, P' = W (a^2 - U) = (sc^6 / 16) P:
// 7 fp64 instructions (2 DADD, 2 DMUL, 3 DFMA) where the image loop needs 10, and the
// constant factor is folded into the log table (a.prod_log_off). a^2 - U cancels where a
// pair is close to a +-d image (absolute error ~3e-15 against 4 delta^2 at relative distance
// delta), so only tile pairs whose bounding boxes keep every pair at least d / 8 from both
// images take it (relative error <= 5e-14 in P, i.e. in the pair's log; the tier's budget
// is 3e-13): prod_mode(). Every other tile pair runs the image loop on the same scaled
// points -- (t - s) - shift scales exactly by a power of two, so its values and its exact
// zeros are those of the unscaled points (apply.cpp:534).
// PROD_ = 1: as above. PROD_ = 2 (any other period): the same on the unscaled binned points,
// with a = W + d^2 and b = a^2 - 4 d^2 U (one more multiplication per image row) and the
// cell's own shifts in the image loop.
template <bool LOWP_, bool CLOG = false, int PROD_ = 0>  // CLOG: coarse table log (eps >= 1e-10, a.coarse_log)
struct SymLaplace {
  static constexpr int NW = 1, NV = 1, NACC = 1, NOUT = 1, TPT = PROD_ ? PWB_SYM_PROD_TPT : PWB_SYM_LAPLACE_TPT,
                       CPT = PROD_ ? PWB_SYM_PROD_CPT : PWB_SYM_LAPLACE_CPT,
                       CHUNK = PROD_ ? PWB_SYM_PROD_ITEM_SOURCES / (128 * PWB_SYM_PROD_CPT)
                                     : 8 * PWB_SYM_LAPLACE_TPT / PWB_SYM_LAPLACE_CPT,  // 4096 sources per item
                       MINB = PROD_ ? PWB_SYM_PROD_MINB : PWB_SYM_LAPLACE_MINB,
                       UNROLL = PROD_ ? PWB_SYM_PROD_UNROLL : PWB_SYM_LAPLACE_UNROLL;
  static constexpr bool FAST = true, LOWP = LOWP_, EXP_TAB = false, CULL = false, PROD = PROD_ != 0,
                        SCALED = PROD_ == 1;  // points pre-scaled to period 2
  static constexpr int THREADS = PROD_ ? PWB_SYM_PROD_THREADS : 128;
  static constexpr bool LOG_SEED = PROD_ && PWB_SYM_PROD_SEED;  // table type: pwk::LogR instead of pwk::LogT
  static_assert(!PROD || LOWP_, "the product form belongs to the reduced tiers");
  // product form of a separated tile pair (see above); dx, dy in the tile's units. NROW == 3
  // (unskewed doubly periodic cells): every image row at (n - 1) eta has the same closed
  // form with its own ry; 19 fp64 instructions for the 9 images where the image loop needs 26.
  template <int NROW, class LK, class B>
  __device__ __forceinline__ static void values_prod(double* V, double dx, double dy, const NearArgs& a, const LK& K,
                                                     B& bad) {
    const double U = dx * dx;
    double P = 1.0;
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = (NROW == 1 || n == 1) ? dy : dy - (n == 0 ? -a.prod_eta : a.prod_eta);
      const double W = fma(ry, ry, U);
      const double aa = SCALED ? fma(W, 0.25, 1.0) : W + a.prod_d2;
      const double b = SCALED ? fma(aa, aa, -U) : fma(aa, aa, -(a.prod_4d2 * U));
      P = n == 0 ? W * b : P * (W * b);
    }
    V[0] = pwk::log_fast(P, K, bad);
  }
  // 128-point column tiles under the 512-point row tile: the staged sources and per-warp
  // column partials take 7 KB, so the conflict-free 8-replica log table (16 KB) and 7
  // blocks per SM fit
  static constexpr int LOG_REPL = PROD_ ? PWB_SYM_PROD_REPL : (CLOG ? PWB_SYM_CLOG_REPL : PWB_SYM_LAPLACE_REPL),
                       LOG_BITS = CLOG ? PWB_SYM_CLOG_TAB : pwk::kLogTabBits;  // 256 x 4 x 16 B = 16 KB
  template <int NXI, int NROW, bool USK, class LK, class B>
  __device__ __forceinline__ static void values_fast(double* V, double dx, double dy, const NearArgs& a,
                                                     const LK& K, B& bad) {
    double ry2[NROW];
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = !SCALED ? row_dy<NXI, NROW>(dy, a, n)
                                : ((NROW == 1 || n == 1) ? dy : dy - (n == 0 ? -a.prod_eta : a.prod_eta));
      ry2[n] = ry * ry;
    }
    if constexpr (SCALED) {
      // scaled points: column shifts -2, 0, 2, rows at (n - 1) eta; per row the product is
      // sc^6 P_row = 16 P'_row, the table expects P'
      static_assert(!SCALED || (NXI == 3 && (NROW == 1 || NROW == 3)), "image rows of three");
      const double xm = dx + 2.0, xp = dx - 2.0;
      double P = NROW == 1 ? 0x1p-4 : 0x1p-12;
#pragma unroll
      for (int n = 0; n < NROW; ++n) P *= fma(xm, xm, ry2[n]) * (fma(dx, dx, ry2[n]) * fma(xp, xp, ry2[n]));
      V[0] = pwk::log_fast(P, K, bad);
      return;
    }
    double P = 1.0;
#pragma unroll
    for (int n = 0; n < NROW; ++n)
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW, USK>(dx, a, n, m);
        P *= fma(rx, rx, ry2[n]);
      }
    V[0] = pwk::log_fast(P, K, bad);
  }
  template <int NXI, int NROW>
  __device__ __noinline__ static void values(double* V, double dx, double dy, const NearArgs& a, int& flag) {
    double L = 0.0;
    for (int n = 0; n < NROW; ++n)
      for (int m = 0; m < NXI; ++m) {
        // SCALED: scaled points, shift m d * sc = 2 (m - 1); each image's log carries ln sc^2
        const double rx = SCALED ? dx - 2.0 * (m - 1) : img_dx<NXI, NROW>(dx, a, n, m);
        const double ry = SCALED ? (NROW == 1 ? dy : dy - a.prod_eta * (n - 1)) : row_dy<NXI, NROW>(dy, a, n);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        L += pwk::log_r2_safe(rx, ry);
        if (SCALED) L -= a.prod_ln_sc2;
      }
    V[0] = L;
  }
  __device__ __forceinline__ static void row(double* acc, const double* V, const double* w) {
    acc[0] = fma(w[0], V[0], acc[0]);
  }
  __device__ __forceinline__ static void col(double* acc, const double* V, const double* w) {
    acc[0] = fma(w[0], V[0], acc[0]);
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0] * (-1.0 / (4.0 * pwk::kPi));
  }
};

template <bool GRAD, bool LOWP_, bool COARSE = false>
struct SymModHelm {  // COARSE: eps >= 1e-9 Bessel tier (pw_math.cuh k01_asym)
  static constexpr int NW = 1, NV = GRAD ? 3 : 1, NACC = NV, NOUT = NV, TPT = PWB_SYM_MH_TPT, CHUNK = 16, MINB = 0,
                       UNROLL = 1;
  static constexpr bool FAST = false, LOWP = LOWP_;
  static constexpr bool EXP_TAB = LOWP_;  // k01_tile<true, .> reads the shared exp table
  static constexpr bool CULL = true;      // per-tile image mask from bounding boxes (see near_sym_body)
  static constexpr bool CHEB = !GRAD;     // regime 3: per-tile-pair Chebyshev K0 (pw_math.cuh cheb_fit_k0)
  static constexpr bool PROD = false, LOG_SEED = false;
  static constexpr int THREADS = 128;
  template <int NROW, class LK, class B>
  __device__ __forceinline__ static void values_prod(double*, double, double, const NearArgs&, const LK&, B&) {}
  static constexpr int CPT = TPT, LOG_REPL = pwk::kLogTabReplicas, LOG_BITS = pwk::kLogTabBits;
  template <int NXI, int NROW, bool USK, class LK, class B>
  __device__ __forceinline__ static void values_fast(double*, double, double, const NearArgs&, const LK&, B&) {}
  // mask: bit n * NXI + m set for the images that may hold a pair with beta r < 64 in this
  // tile pair (block-uniform, so the skips are uniform branches)
  template <int NXI, int NROW>
  __device__ __forceinline__ static void values(double* V, double dx, double dy, const NearArgs& a, int& flag,
                                                unsigned mask) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V[v] = 0.0;
    // rows rolled, image columns unrolled by kSymMhUnrollM: the Bessel body is long (one
    // copy per image bloated the instantiations ~10x in code size and compile time), but
    // a few independent chains per thread are needed to hide its latency
#pragma unroll 1
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
      const double ry2 = ry * ry;
#pragma unroll kSymMhUnrollM
      for (int m = 0; m < NXI; ++m) {
        if (!((mask >> (n * NXI + m)) & 1u)) continue;
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        const double r2 = fma(rx, rx, ry2);
        if (r2 == 0.0) {
          if (rx == 0.0 && ry == 0.0) {
            if (n * NXI + m != a.id_img) flag = 1;
            continue;
          }
        }
        const double X = a.beta2 * r2;
        if (X < a.xcut2) {
          const pwk::K01 k = pwk::k01_tile<LOWP, GRAD, COARSE>(X);
          V[0] += k.k0;
          if (GRAD) {
            V[1] = fma(k.k1_over_x, rx, V[1]);
            V[2] = fma(k.k1_over_x, ry, V[2]);
          }
        }
      }
    }
  }
  // One image of one pair for the image-outer loop of the off-diagonal tiles: false when
  // the pair contributes nothing (beyond the cut-off, or an exact zero -- skipped in the
  // identity image, flagged in any other, apply.cpp:538-545).
  __device__ __forceinline__ static bool image_value(double* V, double rx, double ry, bool ident,
                                                     const NearArgs& a, int& flag) {
    const double r2 = fma(rx, rx, ry * ry);
    // r2 < 2^-1022 (integer test on the high word) is rare; only an exact zero of the
    // shifted delta is a coincidence
    if (pwk::hi_of(r2) < 0x00100000 && rx == 0.0 && ry == 0.0) {
      if (!ident) flag = 1;
      return false;
    }
    const double X = a.beta2 * r2;
    if (!pwk::lt_hi(X, a.xcut2)) return false;  // xcut2 has a zero low word (engine.cu)
    const pwk::K01 k = pwk::k01_tile<LOWP, GRAD, COARSE>(X);
    V[0] = k.k0;
    if (GRAD) {
      V[1] = k.k1_over_x * rx;
      V[2] = k.k1_over_x * ry;
    }
    return true;
  }
  // Same value as image_value for a pair known to be in asymptotic regime FAR (near if
  // false) and inside the cut-off (pw_math.cuh regime_of): branch-free.
  template <bool FAR>
  __device__ __forceinline__ static void image_fast(double* V, double rx, double ry, const NearArgs& a) {
    const double X = a.beta2 * fma(rx, rx, ry * ry);
    const pwk::K01 k = pwk::k01_asym<LOWP, GRAD, FAR, COARSE>(X);
    V[0] = k.k0;
    if (GRAD) {
      V[1] = k.k1_over_x * rx;
      V[2] = k.k1_over_x * ry;
    }
  }
  __device__ __forceinline__ static void row(double* acc, const double* V, const double* w) {
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = fma(w[0], V[v], acc[v]);
  }
  __device__ __forceinline__ static void col(double* acc, const double* V, const double* w) {
    acc[0] = fma(w[0], V[0], acc[0]);
    if (GRAD) {  // the gradient kernel is odd in r
      acc[1] = fma(-w[0], V[1], acc[1]);
      acc[2] = fma(-w[0], V[2], acc[2]);
    }
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs& a, double* out) {
    out[0] = acc[0] * (1.0 / (2.0 * pwk::kPi));
    if (GRAD) {
      const double gs = -a.beta2 / (2.0 * pwk::kPi);
      out[1] = acc[1] * gs;
      out[2] = acc[2] * gs;
    }
  }
};

// Stokeslet: V = (log prod r2, Txx, Txy, Tyy [, Px, Py]) with T = sum r r^T / r^2,
// P = sum r / r^2 (pressurelet, odd).
// PROD (no pressure, unskewed 3 x 3 images, binned points pre-scaled by a.prod_sc = 2 / d):
// each image row in closed form. With U = dX^2, W = U + ry^2 (the middle image's r^2),
// a = W / 4 + 1, b = a^2 - U (= r-^2 r+^2 / 16) the row's three images give
//   sum 1/r^2  = (2 b + a W) / (2 W b),     sum rx/r^2 = dX (2 b + (a - 2) W) / (2 W b),
// so one reciprocal (of 2 W b, which is also the row's factor of the log's product) serves
// three images: 17 fp64 instructions per row where the image loop needs 22. The same
// cancellation in b as the Laplace product form, the same per-tile-pair rule (prod_mode).
// PROD_ = 2 (a period that is not a power of two): unscaled points, A = W + d^2,
// B = A^2 - 4 d^2 U, sums (B + 2 A W) / (W B) and dX (B + 2 (A - 2 d^2) W) / (W B).
template <bool PRESSURE, bool LOWP_, bool CLOG = false, int PROD_ = 0>  // CLOG: coarse table log (eps >= 1e-10)
struct SymStokes {
  static_assert(!PROD_ || (!PRESSURE && LOWP_), "the product form: velocity only, reduced tiers");
  // Without pressure the tile carries (a, Txy, b) with a = L/2 - Txx, b = L/2 - Tyy and
  // accumulates the two velocity components directly (u_x ~ a f_x - Txy f_y, u_y ~
  // b f_y - Txy f_x): 4 fp64 per side instead of 6 and half the column partials. With
  // pressure: (L, Txx, Txy, Tyy, Px, Py) into (L f, T f, P.f).
  static constexpr int NW = 2, NV = PRESSURE ? 6 : 3, NACC = PRESSURE ? 5 : 2, NOUT = PRESSURE ? 3 : 2,
                       TPT = PWB_SYM_STOKES_TPT, CPT = PWB_SYM_STOKES_CPT < PWB_SYM_STOKES_TPT ? PWB_SYM_STOKES_CPT
                                                                                                : PWB_SYM_STOKES_TPT,
                       CHUNK = 32 / CPT, MINB = PWB_SYM_STOKES_MINB, UNROLL = PWB_SYM_STOKES_UNROLL,
                       LOG_REPL = pwk::kLogTabReplicas, LOG_BITS = CLOG ? PWB_SYM_CLOG_TAB : pwk::kLogTabBits;
  static constexpr bool FAST = true, LOWP = LOWP_, EXP_TAB = false, CULL = false, PROD = PROD_ != 0,
                        SCALED = PROD_ == 1, LOG_SEED = false;
  static constexpr int THREADS = 128;
  template <int NROW, class LK, class B>
  __device__ __forceinline__ static void values_prod(double* V, double dx, double dy, const NearArgs& a, const LK& K,
                                                     B& bad) {
    if constexpr (PROD_) {
      const double U = dx * dx;
      double P = 1.0, tyy = 0.0, txyq = 0.0;
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const double ry = n == 1 ? dy : dy - (n == 0 ? -a.prod_eta : a.prod_eta);  // (dy) - shift, shift = (n - 1) eta
        const double ry2 = ry * ry;
        const double W = ry2 + U;
        double Pr, S, Rq;
        if constexpr (SCALED) {
          const double aa = fma(W, 0.25, 1.0);
          const double b = fma(aa, aa, -U);
          const double b2 = b + b;
          Pr = W * b2;  // 2 W b = r0^2 r-^2 r+^2 / 8
          const double inv = pwk::rcp_tier<LOWP>(Pr);
          S = fma(aa, W, b2) * inv;         // sum_m 1 / r^2
          Rq = fma(aa - 2.0, W, b2) * inv;  // sum_m rx / r^2, over dX
        } else {
          const double A = W + a.prod_d2;
          const double B = fma(A, A, -(a.prod_4d2 * U));
          const double W2 = W + W;
          Pr = W * B;  // r0^2 r-^2 r+^2
          const double inv = pwk::rcp_tier<LOWP>(Pr);
          S = fma(W2, A, B) * inv;
          Rq = fma(W2, A - 2.0 * a.prod_d2, B) * inv;
        }
        if (n == 0) {
          P = Pr;
          tyy = ry2 * S;
          txyq = ry * Rq;
        } else {
          P *= Pr;
          tyy = fma(ry2, S, tyy);
          txyq = fma(ry, Rq, txyq);
        }
      }
      const double L = pwk::log_fast(P, K, bad);  // SCALED: the table carries ln(512 / sc^18)
      V[0] = fma(0.5, L, tyy - 9.0);  // L/2 - Txx, Txx = 9 - Tyy
      V[1] = dx * txyq;
      V[2] = fma(0.5, L, -tyy);
    }
  }
  template <int NXI, int NROW, bool USK, class LK, class B>
  __device__ __forceinline__ static void values_fast(double* V, double dx, double dy, const NearArgs& a,
                                                     const LK& K, B& bad) {
    // Per image row n (common ry): S_n = sum_m 1/r^2, R_n = sum_m rx/r^2. Then
    //   Tyy = sum_n ry_n^2 S_n, Txx = images - Tyy (rx^2/r^2 + ry^2/r^2 = 1 per image; no
    //   exact zero on this path), Txy = sum_n ry_n R_n, pressurelet (sum_n R_n, sum_n ry_n S_n):
    // two fp64 instructions per image besides the reciprocal, instead of three.
    // SCALED (scaled points, period 2, rows at -eta, 0, eta in the tile's units): the product
    // is sc^18 P, the table expects P / 512 of it
    double P = SCALED ? 0x1p-9 : 1.0, tyy = 0.0, txy = 0.0, px = 0.0, py = 0.0;
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = SCALED ? (n == 1 ? dy : dy - (n == 0 ? -a.prod_eta : a.prod_eta)) : row_dy<NXI, NROW>(dy, a, n);
      const double ry2 = ry * ry;
      double S = 0.0, R = 0.0;
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = SCALED ? (m == 1 ? dx : dx - 2.0 * (m - 1)) : img_dx<NXI, NROW, USK>(dx, a, n, m);
        const double r2 = fma(rx, rx, ry2);
        P *= r2;
        const double inv = pwk::rcp_tier<LOWP>(r2);
        if (m == 0) {
          S = inv;
          R = rx * inv;
        } else {
          S += inv;
          R = fma(rx, inv, R);
        }
      }
      if (n == 0) {
        tyy = ry2 * S;
        txy = ry * R;
      } else {
        tyy = fma(ry2, S, tyy);
        txy = fma(ry, R, txy);
      }
      if (PRESSURE) {
        px += R;
        py = fma(ry, S, py);
      }
    }
    const double L = pwk::log_fast(P, K, bad);
    if (PRESSURE) {
      V[0] = L;
      V[1] = static_cast<double>(NXI * NROW) - tyy;
      V[2] = txy;
      V[3] = tyy;
      V[4] = px;
      V[5] = py;
    } else {
      V[0] = fma(0.5, L, tyy - static_cast<double>(NXI * NROW));  // L/2 - Txx, Txx = images - Tyy
      V[1] = txy;
      V[2] = fma(0.5, L, -tyy);
    }
  }
  template <int NXI, int NROW>
  __device__ __noinline__ static void values(double* V, double dx, double dy, const NearArgs& a, int& flag) {
    double L = 0.0, txx = 0.0, txy = 0.0, tyy = 0.0, px = 0.0, py = 0.0;
    for (int n = 0; n < NROW; ++n)
      for (int m = 0; m < NXI; ++m) {
        // SCALED: scaled points (shifts 2 (m - 1), (n - 1) eta in the tile's units); the tensor
        // terms do not depend on the scale, each image's log carries ln sc^2
        const double rx = SCALED ? dx - 2.0 * (m - 1) : img_dx<NXI, NROW>(dx, a, n, m);
        const double ry = SCALED ? dy - a.prod_eta * (n - 1) : row_dy<NXI, NROW>(dy, a, n);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        const double r2 = fma(rx, rx, ry * ry);
        L += pwk::log_r2_safe(rx, ry);
        if (SCALED) L -= a.prod_ln_sc2;
        txx += rx * rx / r2;
        txy += rx * ry / r2;
        tyy += ry * ry / r2;
        px += rx / r2;
        py += ry / r2;
      }
    if (PRESSURE) {
      V[0] = L;
      V[1] = txx;
      V[2] = txy;
      V[3] = tyy;
      V[4] = px;
      V[5] = py;
    } else {
      V[0] = fma(0.5, L, -txx);
      V[1] = txy;
      V[2] = fma(0.5, L, -tyy);
    }
  }
  // PRESSURE: acc = (L fx, L fy, (T f)_x, (T f)_y, P.f); else acc = (a fx - Txy fy, b fy - Txy fx)
  __device__ __forceinline__ static void contract(double* acc, const double* V, const double* w, double sgn) {
    if (PRESSURE) {
      acc[0] = fma(V[0], w[0], acc[0]);
      acc[1] = fma(V[0], w[1], acc[1]);
      acc[2] = fma(V[1], w[0], fma(V[2], w[1], acc[2]));
      acc[3] = fma(V[2], w[0], fma(V[3], w[1], acc[3]));
      acc[4] = fma(sgn * V[4], w[0], fma(sgn * V[5], w[1], acc[4]));
    } else {
      acc[0] = fma(V[0], w[0], fma(-V[1], w[1], acc[0]));
      acc[1] = fma(V[2], w[1], fma(-V[1], w[0], acc[1]));
    }
  }
  __device__ __forceinline__ static void row(double* acc, const double* V, const double* w) {
    contract(acc, V, w, 1.0);
  }
  __device__ __forceinline__ static void col(double* acc, const double* V, const double* w) {
    contract(acc, V, w, -1.0);
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    const double c = -1.0 / (4.0 * pwk::kPi);
    if (PRESSURE) {
      out[0] = c * fma(0.5, acc[0], -acc[2]);
      out[1] = c * fma(0.5, acc[1], -acc[3]);
      out[2] = acc[4] * (1.0 / (2.0 * pwk::kPi));
    } else {
      out[0] = c * acc[0];
      out[1] = c * acc[1];
    }
  }
};

// ---------------------------------------------------------------- the kernel
struct SymArgs {
  NearArgs a;
  int nb;                  // number of row tiles (kT * TPT points)
  int ncb;                 // number of column tiles (kT * CPT points)
  int chunk;                   // column tiles per work item
  const long long* row_start;  // [nb + 1] first work item of each row tile (int64: items grow as n^2)
  unsigned long long* fx;      // fixed-point accumulators [n][nout][3]
  long long item0;             // first work item of this launch (multi-GPU item ranges, 2^31-block chunks)
};

template <class K>
__device__ __forceinline__ void load_w(const NearArgs& a, size_t j, bool live, double* w) {
  if (K::NW == 1) {
    w[0] = live ? a.q[j] : 0.0;
  } else {
    const double2 v = live ? a.vec[j] : make_double2(0.0, 0.0);
    w[0] = v.x;
    w[K::NW > 1 ? 1 : 0] = v.y;
  }
}

template <class K, int NXI, int NROW>
__device__ __forceinline__ void call_values(double* V, double dx, double dy, const NearArgs& a, int& flag,
                                            unsigned mask) {
  if constexpr (K::CULL)
    K::template values<NXI, NROW>(V, dx, dy, a, flag, mask);
  else
    K::template values<NXI, NROW>(V, dx, dy, a, flag);
}

// Images whose every (target, source) pair between the row box and the column box has
// beta^2 r^2 >= xcut2 get their bit cleared: the per-pair test would skip all of them.
// The box gap is a lower bound of |(t - s) - shift| per axis; the 1e-4 margin covers
// its rounding, so the mask never drops a pair the per-pair test would keep.
template <int NXI, int NROW>
__device__ __forceinline__ unsigned image_mask(const double* rb, const double* cb, const NearArgs& a) {
  unsigned mask = 0;
#pragma unroll
  for (int img = 0; img < NXI * NROW; ++img) {
    double lo, hi;
    image_xrange(rb, cb, a.shx[img], a.shy[img / NXI], a.beta2, lo, hi);
    if (lo * 0.9999 < a.xcut2) mask |= 1u << img;
  }
  return mask;
}

// Product-form tiles (SymLaplace / SymStokes PROD), per tile pair from the row box and the
// column box (xmin, -xmax, ymin, -ymax; `period` is 2 for the scaled tiles and d for the
// unscaled ones, the image rows sit at (n - 1) eta):
//   0  some pair may come within period / 8 of an image of the +period or the -period
//      column in both x and y: the image loop;
//   1  every pair stays clear of those images: the product form;
//   2  and no image can coincide with a pair at all (the boxes are apart by more than
//      2^-40 periods around every image), so every product -- down to 2^-276 d^18 for nine
//      images, d within 2^+-30 in the unscaled form -- is a normal number: the product form
//      without the exponent check and without the saved row sums of the careful redo.
template <int NROW>
__device__ __forceinline__ int prod_mode(const double* tb, const double* sb, double eta, double period) {
  const double xlo = tb[0] + sb[1], xhi = -tb[1] - sb[0];  // range of t.x - s.x
  const double ylo = tb[2] + sb[3], yhi = -tb[3] - sb[2];
  auto gap = [](double lo, double hi, double c) { return lo > c ? lo - c : (hi < c ? c - hi : 0.0); };
  const double gx0 = gap(xlo, xhi, 0.0);
  const double gxs = fmin(gap(xlo, xhi, period), gap(xlo, xhi, -period));  // to the nearer side column
  int mode = 2;
#pragma unroll
  for (int n = 0; n < NROW; ++n) {
    const double gy = gap(ylo, yhi, NROW == 1 ? 0.0 : (n - 1) * eta);
    if (!(fmax(gxs, gy) >= 0.125 * period)) return 0;
    if (!(fmax(gx0, gy) > 0x1p-40 * period)) mode = 1;
  }
  return mode;
}

template <class K, int NXI, int NROW, bool USK>
__device__ __forceinline__ void near_sym_body(const SymArgs& S) {
  constexpr int TPT = K::TPT;
  constexpr int kT = K::THREADS, kWarps = kT / 32;
  constexpr int TILE = kT * TPT;          // row tile: the block's targets
  constexpr int CT = kColUnit * K::CPT;   // column tile: the sources staged per step
  constexpr int R = TILE / CT;        // column tiles per row tile
  static_assert(TILE % CT == 0 && (CT & (CT - 1)) == 0, "column tile must divide the row tile");
  const NearArgs& a = S.a;
  __shared__ double s_x[CT], s_y[CT], s_w[K::NW][CT];
  __shared__ double s_col[kWarps][K::NACC][CT];
  __shared__ double s_keep[PWB_SYM_KEEP_SMEM && K::FAST ? TPT * K::NACC : 1][PWB_SYM_KEEP_SMEM && K::FAST ? kT : 1];

  // work item -> (row tile I, first column tile)
  const long long item = S.item0 + static_cast<long long>(blockIdx.x);
  int lo = 0, hi = S.nb;  // row_start[I] <= item < row_start[I+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (S.row_start[mid] <= item)
      lo = mid;
    else
      hi = mid;
  }
  const int I = lo;
  const int J0 = I * R + static_cast<int>(item - S.row_start[I]) * S.chunk;
  const int J1 = min(S.ncb, J0 + S.chunk);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t n = a.nt;
  double tx[TPT], ty[TPT], tw[TPT][K::NW], racc[TPT][K::NACC];
  bool live[TPT];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const size_t l = static_cast<size_t>(I) * TILE + tid + k * kT;
    live[k] = l < n;
    const double2 p = live[k] ? a.tgt[l] : make_double2(0.0, 0.0);  // dead: origin, weight 0
    tx[k] = p.x;
    ty[k] = p.y;
    load_w<K>(a, l, live[k], tw[k]);
#pragma unroll
    for (int c = 0; c < K::NACC; ++c) racc[k][c] = 0.0;
  }
  int flag = 0;
  // log constants in registers; the reduced tier's log table in shared memory
  constexpr size_t kTileSmem = sizeof(double) * (static_cast<size_t>(CT) * (2 + K::NW) + kWarps * K::NACC * CT);
  constexpr int kRepl = K::LOG_REPL, kBits = K::LOG_BITS;
  constexpr size_t kTabEntry = K::LOG_SEED ? sizeof(double) : sizeof(double2);
  constexpr size_t kTabSmem = kTabEntry * (size_t{1} << pwk::tab_bits(kBits)) * kRepl;
  constexpr bool kTab = K::FAST && K::LOWP && PWB_SYM_LOG_TABLE && kTileSmem + kTabSmem <= 48 * 1024;
  __shared__ double2 s_lt[kTab ? kTabSmem / sizeof(double2) : 1];
  using LKT = std::conditional_t<kTab,
                                 std::conditional_t<K::LOG_SEED, pwk::LogR<kRepl, kBits>, pwk::LogT<kRepl, kBits>>,
                                 pwk::LogK<K::LOWP>>;
  LKT LK;
  if constexpr (kTab && K::LOG_SEED) {
    // visible after the first __syncthreads of the tile loop
    pwk::log_seed_fill<kRepl, kBits>(reinterpret_cast<double*>(s_lt), tid, kT, K::PROD ? a.prod_log_off : 0.0);
    LK = pwk::log_seed_consts<kRepl, kBits>(reinterpret_cast<const double*>(s_lt), lane);
  } else if constexpr (kTab) {
    // visible after the first __syncthreads of the tile loop
    pwk::log_tab_fill<kRepl, kBits>(s_lt, tid, kT, K::PROD ? a.prod_log_off : 0.0);
    LK = pwk::log_tab_consts<kRepl, kBits>(s_lt, lane);
  } else if constexpr (K::FAST) {
    LK = pwk::log_consts<K::LOWP>();
  }
  if constexpr (K::EXP_TAB) pwk::exp_tab_fill();  // visible after the first __syncthreads of the tile loop
  // screened kernels: bounding boxes of the row tile and of each column tile -> image mask
  constexpr bool kBoxes = K::CULL || K::PROD;  // PROD: which tile pairs may take the product form
  static_assert(!K::PROD || kTab, "the product form's constant factor lives in the log table");
  __shared__ double s_rbox[kBoxes ? kWarps : 1][4], s_cbox[kBoxes ? kWarps : 1][4];
  if constexpr (kBoxes) {
    double b[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
    for (int k = 0; k < TPT; ++k)
      if (live[k]) {
        b[0] = fmin(b[0], tx[k]);
        b[1] = fmin(b[1], -tx[k]);
        b[2] = fmin(b[2], ty[k]);
        b[3] = fmin(b[3], -ty[k]);
      }
    warp_box_store(b[0], b[1], b[2], b[3], lane, s_rbox[warp]);  // read after the tile loop's syncs
  }

  for (int J = J0; J < J1; ++J) {
    const size_t jbase = static_cast<size_t>(J) * CT;
    __syncthreads();
    double cb[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    for (int i = tid; i < CT; i += kT) {
      const size_t j = jbase + i;
      const bool lv = j < n;
      const double2 p = lv ? a.src[j] : make_double2(0.0, 0.0);
      s_x[i] = p.x;
      s_y[i] = p.y;
      if (kBoxes && lv) {
        cb[0] = fmin(cb[0], p.x);
        cb[1] = fmin(cb[1], -p.x);
        cb[2] = fmin(cb[2], p.y);
        cb[3] = fmin(cb[3], -p.y);
      }
      double w[K::NW];
      load_w<K>(a, j, lv, w);
#pragma unroll
      for (int c = 0; c < K::NW; ++c) s_w[c][i] = w[c];
#pragma unroll
      for (int c = 0; c < K::NACC; ++c)
#pragma unroll
        for (int wv = 0; wv < kWarps; ++wv) s_col[wv][c][i] = 0.0;
    }
    if constexpr (kBoxes) warp_box_store(cb[0], cb[1], cb[2], cb[3], lane, s_cbox[warp]);
    __syncthreads();
    unsigned mask = ~0u;
    double rb[4], cbx[4];
    if (kBoxes && (K::PROD || a.cull)) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if constexpr (kWarps == 4) {
          rb[c] = fmin(fmin(s_rbox[0][c], s_rbox[1][c]), fmin(s_rbox[2][c], s_rbox[3][c]));
          cbx[c] = fmin(fmin(s_cbox[0][c], s_cbox[1][c]), fmin(s_cbox[2][c], s_cbox[3][c]));
        } else {
          rb[c] = s_rbox[0][c];
          cbx[c] = s_cbox[0][c];
#pragma unroll
          for (int wv = 1; wv < kWarps; ++wv) {
            rb[c] = fmin(rb[c], s_rbox[wv][c]);
            cbx[c] = fmin(cbx[c], s_cbox[wv][c]);
          }
        }
      }
    }
    if (K::CULL && a.cull) {
      mask = image_mask<NXI, NROW>(rb, cbx, a);
      if (mask == 0u) continue;  // block-uniform: no pair of this tile pair is in range
    }
    if (J < (I + 1) * R) {  // inside the row tile: one-sided (self pairs live here)
      if constexpr (K::FAST) {
        // Fast one-sided sweep: every ordered pair once with the branch-free pair values; a
        // thread's own point (identity image skipped, apply.cpp:538-545) takes the other
        // images' values at the pure shifts, which the careful evaluation of a zero delta
        // returns (once per tile). A duplicate point or an image coincidence makes a product
        // vanish and sends the tile to the careful sweep below. The careful sweep alone is
        // ~10x slower per pair: these tiles are ~0.1 % of the pairs, but one such work item
        // per row tile ran 5-7 ms and sat at the end of every rank's item range (8-rank near
        // efficiency of c4 0.93, r3p).
        double Vself[K::NV];
        {
          int f0 = 0;
          call_values<K, NXI, NROW>(Vself, 0.0, 0.0, a, f0, mask);
        }
        double keepd[TPT][K::NACC];
#pragma unroll
        for (int k = 0; k < TPT; ++k)
#pragma unroll
          for (int c = 0; c < K::NACC; ++c) keepd[k][c] = racc[k][c];
        using BadD = std::conditional_t<kTab, unsigned, int>;
        BadD badd = 0;
        const bool dprod = K::PROD && prod_mode<NROW>(rb, cbx, a.prod_eta, a.prod_period) >= 1;  // block-uniform
        const size_t l0 = static_cast<size_t>(I) * TILE + tid;
        auto diag_loop = [&](auto prod) {
#pragma unroll 2
          for (int i = 0; i < CT; ++i) {
            const double sx = s_x[i], sy = s_y[i];
            double w[K::NW];
#pragma unroll
            for (int c = 0; c < K::NW; ++c) w[c] = s_w[c][i];
#pragma unroll
            for (int k = 0; k < TPT; ++k) {
              double V[K::NV];
              BadD b1 = 0;
              if constexpr (decltype(prod)::value)
                K::template values_prod<NROW>(V, tx[k] - sx, ty[k] - sy, a, LK, b1);
              else
                K::template values_fast<NXI, NROW, USK>(V, tx[k] - sx, ty[k] - sy, a, LK, b1);
              const bool self = jbase + i == l0 + static_cast<size_t>(k) * kT;
              if (!self) badd = max(badd, b1);
#pragma unroll
              for (int c = 0; c < K::NV; ++c) V[c] = self ? Vself[c] : V[c];
              K::row(racc[k], V, w);
            }
          }
        };
        if (dprod)
          diag_loop(std::true_type{});
        else
          diag_loop(std::false_type{});
        if (!__syncthreads_or(pwk::log_bad(LK, badd))) continue;
#pragma unroll
        for (int k = 0; k < TPT; ++k)
#pragma unroll
          for (int c = 0; c < K::NACC; ++c) racc[k][c] = keepd[k][c];
      }
      for (int i = 0; i < CT; ++i) {
        const double sx = s_x[i], sy = s_y[i];
        double w[K::NW];
#pragma unroll
        for (int c = 0; c < K::NW; ++c) w[c] = s_w[c][i];
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          double V[K::NV];
          call_values<K, NXI, NROW>(V, tx[k] - sx, ty[k] - sy, a, flag, mask);
          K::row(racc[k], V, w);
        }
      }
      continue;
    }
    bool careful = !K::FAST;
    if constexpr (K::CULL) {
      // Screened tiles, off-diagonal: image-outer order. The image's shift is loop-invariant
      // and its mask bit is tested once per tile pair, the inner loop is one K0 (K1) per
      // (target, source) -- small code, two sources in flight -- and the column partials
      // take one shared-memory update per (image, source).
#pragma unroll 1
      for (int img = 0; img < NXI * NROW; ++img) {
        if (!((mask >> img) & 1u)) continue;
        const double shx = a.shx[img], shy = a.shy[img / NXI];
        const bool ident = img == a.id_img;
        int regime = 0;  // per-pair dispatch unless the boxes pin the whole tile pair
        pwk::ChebFit<kChebMax> cf;
        if (a.cull) {
          double lo, hi;
          image_xrange(rb, cbx, shx, shy, a.beta2, lo, hi);
          regime = pwk::regime_of(lo, hi, a.xcut2);
          if constexpr (K::CHEB) {
            // regime 3: the tile pair's s = r^2 interval is short enough for one fitted
            // polynomial (block-uniform: every warp fits the same interval identically).
            // x >= 0.5 keeps it clear of the log singularity and of any exact zero.
            if (a.cheb_tol > 0.0 && lo * 0.9999 > 0.25) {
              pwk::cheb_fit_k0(lo * 0.9999, hi * 1.0001, a.beta2, a.inv_beta2, a.cheb_tol, cf);
              if (cf.deg) regime = 3;
            }
          }
        }
        auto sweep = [&](auto reg, auto cdeg) {
          constexpr int R = decltype(reg)::value;
          constexpr int CD = decltype(cdeg)::value;  // regime 3: the fitted degree
          // regime sweeps (no coincidence possible, X_lo > 4): the shifted targets are formed
          // once per image, (t - shift) - s, one subtraction per coordinate and pair; the
          // per-pair dispatch keeps the reference's association (t - s) - shift
          // (apply.cpp:534), whose exact zeros decide CoincidentSourceTarget
          double txs[TPT], tys[TPT];
#pragma unroll
          for (int k = 0; k < TPT; ++k) {
            txs[k] = tx[k] - shx;
            tys[k] = ty[k] - shy;
          }
          constexpr int kU = R == 0 ? PWB_SYM_MH_GEN_UNROLL : kSymMhSrcUnroll;  // the per-pair dispatch is branchy: less unrolled
#pragma unroll kU
          for (int i = 0; i < CT; ++i) {
            const int jj = (lane + i) & (CT - 1);
            const double sx = s_x[jj], sy = s_y[jj];
            double w[K::NW];
#pragma unroll
            for (int c = 0; c < K::NW; ++c) w[c] = s_w[c][jj];
            double cacc[K::NACC];
#pragma unroll
            for (int c = 0; c < K::NACC; ++c) cacc[c] = 0.0;
#pragma unroll
            for (int k = 0; k < TPT; ++k) {
              double V[K::NV];
              const double rx = R == 0 ? (tx[k] - sx) - shx : txs[k] - sx;
              const double ry = R == 0 ? (ty[k] - sy) - shy : tys[k] - sy;
              if constexpr (R == 0) {
                if (!K::image_value(V, rx, ry, ident, a, flag)) continue;
              } else if constexpr (R == 3) {
                V[0] = pwk::cheb_eval<CD>(cf, rx, ry);
              } else {
                K::template image_fast<R == 2>(V, rx, ry, a);
              }
              K::row(racc[k], V, w);
              K::col(cacc, V, tw[k]);
            }
#pragma unroll
            for (int c = 0; c < K::NACC; ++c) s_col[warp][c][jj] += cacc[c];
          }
        };
        using I0 = std::integral_constant<int, 0>;
        if constexpr (K::CHEB) {
          if (regime == 3) {
            if (cf.deg == 6)
              sweep(std::integral_constant<int, 3>{}, std::integral_constant<int, 6>{});
            else if (cf.deg == 9)
              sweep(std::integral_constant<int, 3>{}, std::integral_constant<int, 9>{});
            else
              sweep(std::integral_constant<int, 3>{}, std::integral_constant<int, kChebMax>{});
            continue;
          }
        }
        if (regime == 2)
          sweep(std::integral_constant<int, 2>{}, I0{});
        else if (regime == 1 && PWB_SYM_MH_NEAR_SWEEP)
          sweep(std::integral_constant<int, 1>{}, I0{});
        else
          sweep(std::integral_constant<int, 0>{}, I0{});
      }
      careful = false;
    }
    // the branch-free sweep of the staged column tile: prod selects the product form of the
    // pair values, `bad` collects the exponent check (a local nobody reads drops it)
    auto fast_loop = [&](auto prod, auto& bad) {
#pragma unroll K::UNROLL
      for (int i = 0; i < CT; ++i) {
        const int jj = (lane + i) & (CT - 1);
        const double sx = s_x[jj], sy = s_y[jj];
        double w[K::NW];
#pragma unroll
        for (int c = 0; c < K::NW; ++c) w[c] = s_w[c][jj];
        double cacc[K::NACC];
#pragma unroll
        for (int c = 0; c < K::NACC; ++c) cacc[c] = 0.0;
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          double V[K::NV];
          // (t - s) - shift as upstream (apply.cpp:534)
          if constexpr (decltype(prod)::value)
            K::template values_prod<NROW>(V, tx[k] - sx, ty[k] - sy, a, LK, bad);
          else
            K::template values_fast<NXI, NROW, USK>(V, tx[k] - sx, ty[k] - sy, a, LK, bad);
          K::row(racc[k], V, w);
          K::col(cacc, V, tw[k]);
        }
#pragma unroll
        for (int c = 0; c < K::NACC; ++c) s_col[warp][c][jj] += cacc[c];
      }
    };
    using BadT = std::conditional_t<kTab, unsigned, int>;  // see pwk::log_bad
    int pmode = 0;
    if constexpr (K::PROD) {
      pmode = prod_mode<NROW>(rb, cbx, a.prod_eta, a.prod_period);  // block-uniform
      // dead rows / columns sit at the origin with weight 0: their products may vanish, so a
      // ragged tile pair keeps the check
      if (pmode == 2 && (static_cast<size_t>(I + 1) * TILE > n || jbase + CT > n)) pmode = 1;
      if (pmode == 2) {
        BadT unchecked = 0;
        fast_loop(std::true_type{}, unchecked);
      }
    }
    if (K::FAST && pmode != 2) {
      // the row sums before this tile, for the careful redo: in shared memory (each thread
      // its own column, no sync needed) when PWB_SYM_KEEP_SMEM, else in registers
      double keep[PWB_SYM_KEEP_SMEM ? 1 : TPT][K::NACC];
#pragma unroll
      for (int k = 0; k < TPT; ++k)
#pragma unroll
        for (int c = 0; c < K::NACC; ++c) {
          if constexpr (PWB_SYM_KEEP_SMEM)
            s_keep[k * K::NACC + c][tid] = racc[k][c];
          else
            keep[k][c] = racc[k][c];
        }
      BadT bad = 0;
      if (K::PROD && pmode == 1)
        fast_loop(std::true_type{}, bad);
      else
        fast_loop(std::false_type{}, bad);
      if (__syncthreads_or(pwk::log_bad(LK, bad))) {  // rare: redo this tile on the careful path
#pragma unroll
        for (int k = 0; k < TPT; ++k)
#pragma unroll
          for (int c = 0; c < K::NACC; ++c) racc[k][c] = PWB_SYM_KEEP_SMEM ? s_keep[k * K::NACC + c][tid] : keep[k][c];
        for (int i = tid; i < CT; i += kT)
#pragma unroll
          for (int c = 0; c < K::NACC; ++c)
#pragma unroll
            for (int wv = 0; wv < kWarps; ++wv) s_col[wv][c][i] = 0.0;
        __syncthreads();
        careful = true;
      }
    }
    if (careful) {
#pragma unroll 1
      for (int i = 0; i < CT; ++i) {
        const int jj = (lane + i) & (CT - 1);
        const double sx = s_x[jj], sy = s_y[jj];
        double w[K::NW];
#pragma unroll
        for (int c = 0; c < K::NW; ++c) w[c] = s_w[c][jj];
        double cacc[K::NACC];
#pragma unroll
        for (int c = 0; c < K::NACC; ++c) cacc[c] = 0.0;
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          double V[K::NV];
          call_values<K, NXI, NROW>(V, tx[k] - sx, ty[k] - sy, a, flag, mask);
          K::row(racc[k], V, w);
          K::col(cacc, V, tw[k]);
        }
#pragma unroll
        for (int c = 0; c < K::NACC; ++c) s_col[warp][c][jj] += cacc[c];
      }
    }
    __syncthreads();
    // column totals of this tile -> fixed point
    for (int i = tid; i < CT; i += kT) {
      const size_t j = jbase + i;
      if (j >= n) continue;
      double acc[K::NACC];
#pragma unroll
      for (int c = 0; c < K::NACC; ++c) {
        double s = 0.0;
#pragma unroll
        for (int wv = 0; wv < kWarps; ++wv) s += s_col[wv][c][i];
        acc[c] = s;
      }
      double o[K::NOUT];
      K::finish(acc, a, o);
#pragma unroll
      for (int c = 0; c < K::NOUT; ++c) fx_add(S.fx + (j * K::NOUT + c) * 3, o[c], a);
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    if (!live[k]) continue;
    const size_t l = static_cast<size_t>(I) * TILE + tid + k * kT;
    double o[K::NOUT];
    K::finish(racc[k], a, o);
#pragma unroll
    for (int c = 0; c < K::NOUT; ++c) fx_add(S.fx + (l * K::NOUT + c) * 3, o[c], a);
  }
  if (flag) atomicOr(a.flag, 1);
}


// K::MINB > 0 caps registers for K::MINB resident blocks per SM (one image row; the 2-D
// image blocks hold more live shifts and get at most 4 -- 80 or 96 regs spill there).
// MINB == 0 keeps ptxas's own allocation (the wider functors).
template <class K, int NXI, int NROW, bool USK>
__global__ void __launch_bounds__(K::THREADS, NROW == 1 ? K::MINB : (K::MINB < 4 ? K::MINB : 4))
    near_sym_kernel_capped(const __grid_constant__ SymArgs S) {
  near_sym_body<K, NXI, NROW, USK>(S);
}

template <class K, int NXI, int NROW, bool USK>
__global__ void __launch_bounds__(K::THREADS) near_sym_kernel(const __grid_constant__ SymArgs S) {
  near_sym_body<K, NXI, NROW, USK>(S);
}

template <class K, int NXI, int NROW, bool USK = false>
void launch_sym_shape(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* row_start_dev,
                      long long* row_start_host, const SymRange& range) {
  constexpr int kT = K::THREADS, TILE = kT * K::TPT, CT = kColUnit * K::CPT, R = TILE / CT;
  const int chunk = K::CHUNK;
  const int nb = static_cast<int>((a.nt + TILE - 1) / TILE);
  const int ncb = static_cast<int>((a.nt + CT - 1) / CT);
  long long items = 0;
  for (int I = 0; I < nb; ++I) {
    row_start_host[I] = items;
    items += (ncb - static_cast<long long>(I) * R + chunk - 1) / chunk;
  }
  row_start_host[nb] = items;
  if (range.total_items) *range.total_items = items;
  if (range.count_only) return;
  const long long b = range.begin < 0 ? 0 : std::min<long long>(range.begin, items);
  const long long e = range.end < 0 ? items : std::min<long long>(range.end, items);
  cuda_check(cudaMemcpyAsync(row_start_dev, row_start_host, (nb + 1) * sizeof(long long), cudaMemcpyHostToDevice, st),
             "row starts");
  const size_t nout = K::NOUT;
  if (range.finish) cuda_check(cudaMemsetAsync(fx, 0, 3 * a.nt * nout * sizeof(unsigned long long), st), "memset fx");
  SymArgs S;
  S.a = a;
  S.nb = nb;
  S.ncb = ncb;
  S.chunk = chunk;
  S.row_start = row_start_dev;
  S.fx = fx;
  void (*kern)(const SymArgs);
  if constexpr (K::MINB > 0)
    kern = near_sym_kernel_capped<K, NXI, NROW, USK>;
  else
    kern = near_sym_kernel<K, NXI, NROW, USK>;
  if (e > b) set_max_carveout(reinterpret_cast<const void*>(kern));
  // grids of at most 2^31 - 1 blocks (items grow as n^2: ~2^31 near n ~ 1e8 for Laplace)
  constexpr long long kMaxGrid = 0x7fffffffLL;
  for (long long i0 = b; i0 < e; i0 += kMaxGrid) {
    S.item0 = i0;
    kern<<<static_cast<unsigned>(std::min(kMaxGrid, e - i0)), kT, 0, st>>>(S);
    count_launches(1);
  }
  if (range.finish) launch_fx_finish(fx, a.nt, a.out0, a.nout0, a.out1, a.nout1, a.out_row, a.fx_maxhi, a.ns, 0, a.flag, st);
}

template <class K>
bool dispatch_sym(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd, long long* rsh,
                  const SymRange& r) {
  if (a.nxi == 3 && a.nrow == 1) return launch_sym_shape<K, 3, 1>(a, st, fx, rsd, rsh, r), true;
  // unskewed 3x3 (c1, c3, c5's cells): the fast tiles form each column's rx once per pair
  if (a.nxi == 3 && a.nrow == 3 && a.unskewed && K::FAST) return launch_sym_shape<K, 3, 3, true>(a, st, fx, rsd, rsh, r), true;
  if (a.nxi == 3 && a.nrow == 3) return launch_sym_shape<K, 3, 3>(a, st, fx, rsd, rsh, r), true;
  if (a.nxi == 5 && a.nrow == 3) return launch_sym_shape<K, 5, 3>(a, st, fx, rsd, rsh, r), true;
  if (a.nxi == 7 && a.nrow == 3) return launch_sym_shape<K, 7, 3>(a, st, fx, rsd, rsh, r), true;
  return false;
}

// per-family entry points (one translation unit each)
bool launch_laplace(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd, long long* rsh,
                    const SymRange& r);
bool launch_modhelm(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd,
                    long long* rsh, const SymRange& r);
bool launch_stokes(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd,
                   long long* rsh, const SymRange& r);

}  // namespace sym
}  // namespace pwb
