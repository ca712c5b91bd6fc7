// Near-image P2P tiles: every near lattice image fused into one launch.
//
// Replaces the reference's per-image double loop
// (/root/reference/proj/src/apply.cpp:481-546, called once per image at :553-554)
// and its pair kernels (kernels.cpp:98-162). One thread owns TPT targets in
// registers; sources stream through shared memory in tiles (all lanes read
// the same source -> broadcast, no bank conflicts); every (target, source)
// pair is evaluated for all NXI x NROW images before moving on, so position
// deltas, strengths and the log are shared across images:
//   * Laplace / Stokeslet log terms: sum_img q log r2_img = q log(prod_img r2_img),
//     one log per (target, source) instead of one per image;
//   * zero-distance semantics of the reference (identity image skips exact
//     zeros, any other image raises CoincidentSourceTarget) are kept exactly:
//     a product that is 0/subnormal/inf falls to a per-image slow path.
// Accumulation is fp64 in registers; with source splits the per-split partial
// sums are combined in fixed order (deterministic for a given launch shape).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "pw_engine.cuh"
#include "pw_math.cuh"
#include "pw_pair.cuh"
#include "near_common.cuh"

#ifndef PWB_MH_SRC_UNROLL
#define PWB_MH_SRC_UNROLL 8  // sources per unrolled step of the screened image-outer sweeps (c2: 2 -> 579 ms, 4 -> 566; r3u/r3v with today's tile: 4 -> 488, 8 -> 467, 12 -> 458, 16 -> 460; with the near sweep 6 / 8 / 12 -> 460 / 455 / 456)
#endif
#ifndef PWB_MH_GEN_UNROLL
#define PWB_MH_GEN_UNROLL 1  // sources per unrolled step of the per-pair-dispatch sweep
#endif
#ifndef PWB_MH_NEAR_SWEEP
#define PWB_MH_NEAR_SWEEP 1  // 1: a tile pair wholly in 2 <= x < 6 gets its own sweep (round 1, unroll 4: 520 ms vs 512 without; r3v at unroll 8: 455 vs 467)
#endif
#ifndef PWB_MH_TPT
#define PWB_MH_TPT 1  // targets per thread of the screened one-sided tiles
#endif
namespace pwb {
namespace {
constexpr int kMhSrcUnroll = PWB_MH_SRC_UNROLL;
}
}  // namespace pwb

namespace pwb {
namespace {

constexpr int kThreads = 128;
#ifndef PWB_NEAR_TILE
#define PWB_NEAR_TILE 256  // sources staged per step of the one-sided tile
#endif
constexpr int kTile = PWB_NEAR_TILE;

// ---------------------------------------------------------------- pair functors
// Each functor: NW strength doubles per source, NACC accumulators per target,
// NOUT output doubles per target, pair<NXI,NROW>(acc, dx, dy, w, args, flag),
// finish(acc, args, out[NOUT]).

template <bool LOWP>
struct Laplace {  // -log|r| / 2pi  (kernels.cpp:102-103)
  static constexpr int NW = 1, NACC = 1, NOUT = 1;
  using Consts = pwk::LogK<LOWP>;  // register-resident log constants (pw_math.cuh)
  __device__ __forceinline__ static Consts consts() { return pwk::log_consts<LOWP>(); }
  template <int NXI, int NROW>
  __device__ __forceinline__ static void pair(double* acc, double dx, double dy, const double* w,
                                              const NearArgs& a, int& flag, const Consts& C) {
    double ry2[NROW];
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
      ry2[n] = ry * ry;
    }
    double P = 1.0;
#pragma unroll
    for (int n = 0; n < NROW; ++n)
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        P *= fma(rx, rx, ry2[n]);
      }
    int bad = 0;
    const double LP = pwk::log_pos_k<LOWP>(P, C, bad);
    if (!bad) {
      acc[0] = fma(w[0], LP, acc[0]);
      return;
    }
    // A self pair (targets == sources) or a duplicate point: the identity image's exact zero
    // is skipped (apply.cpp:536-539) and the other images' product is normally fine -- one
    // log of it. (Without this shortcut every self pair ran the per-image loop below, and the
    // one warp of a block holding the block's self pairs ran it once per source: c1's near
    // tile went 37 -> ~5 us.) Any other exact zero flags the coincidence.
    double Q = 1.0;
    bool other_zero = false;
#pragma unroll
    for (int n = 0; n < NROW; ++n)
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        const double ry = row_dy<NXI, NROW>(dy, a, n);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) other_zero = true;
          continue;
        }
        Q *= fma(rx, rx, ry * ry);
      }
    if (other_zero) flag = 1;
    int bad2 = 0;
    const double LQ = pwk::log_pos_k<LOWP>(Q, C, bad2);
    if (!bad2 && !other_zero) {
      acc[0] = fma(w[0], LQ, acc[0]);
      return;
    }
    double L = 0.0;
#pragma unroll 1
    for (int n = 0; n < NROW; ++n)
#pragma unroll 1
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        const double ry = row_dy<NXI, NROW>(dy, a, n);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        L += pwk::log_r2_safe(rx, ry);
      }
    acc[0] = fma(w[0], L, acc[0]);
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0] * (-1.0 / (4.0 * pwk::kPi));
  }
};

template <bool LOWP, bool COARSE = false>  // COARSE: the coarse Bessel tier (pw_math.cuh k01_asym)
struct ModHelm {  // K0(beta r) / 2pi  (kernels.cpp:104-106)
  static constexpr int NW = 1, NACC = 1, NOUT = 1;
  static constexpr bool EXP_TAB = LOWP;  // k01_tile<true, .> reads the shared exp table
  // one image of one pair (image-outer loop of near_tile_kernel): same semantics as pair()
  static constexpr bool IMAGE_OUTER = true;
  __device__ __forceinline__ static void image(double* acc, double rx, double ry, const double* w, bool ident,
                                               const NearArgs& a, int& flag) {
    const double r2 = fma(rx, rx, ry * ry);
    // r2 < 2^-1022 (integer test on the high word) is rare; only an exact zero of the
    // shifted delta is a coincidence
    if (pwk::hi_of(r2) < 0x00100000 && rx == 0.0 && ry == 0.0) {
      if (!ident) flag = 1;
      return;
    }
    const double X = a.beta2 * r2;
    if (pwk::lt_hi(X, a.xcut2)) acc[0] = fma(w[0], pwk::k01_tile<LOWP, false, COARSE>(X).k0, acc[0]);
  }
  // the same for a pair known to be in asymptotic regime FAR and inside the cut-off
  template <bool FAR>
  __device__ __forceinline__ static void image_fast(double* acc, double rx, double ry, const double* w,
                                                    const NearArgs& a) {
    const double X = a.beta2 * fma(rx, rx, ry * ry);
    acc[0] = fma(w[0], pwk::k01_asym<LOWP, false, FAR, COARSE>(X).k0, acc[0]);
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0] * (1.0 / (2.0 * pwk::kPi));
  }
};

template <bool LOWP, bool COARSE = false>
struct ModHelmGrad {  // u and grad u = -(beta/2pi) K1(beta r) r_vec / r
  static constexpr int NW = 1, NACC = 3, NOUT = 3;
  static constexpr bool EXP_TAB = LOWP;
  static constexpr bool IMAGE_OUTER = true;
  __device__ __forceinline__ static void image(double* acc, double rx, double ry, const double* w, bool ident,
                                               const NearArgs& a, int& flag) {
    const double r2 = fma(rx, rx, ry * ry);
    // r2 < 2^-1022 (integer test on the high word) is rare; only an exact zero of the
    // shifted delta is a coincidence
    if (pwk::hi_of(r2) < 0x00100000 && rx == 0.0 && ry == 0.0) {
      if (!ident) flag = 1;
      return;
    }
    const double X = a.beta2 * r2;
    if (pwk::lt_hi(X, a.xcut2)) {
      const pwk::K01 k = pwk::k01_tile<LOWP, true, COARSE>(X);
      acc[0] = fma(w[0], k.k0, acc[0]);
      const double g = w[0] * k.k1_over_x;
      acc[1] = fma(g, rx, acc[1]);
      acc[2] = fma(g, ry, acc[2]);
    }
  }
  template <bool FAR>
  __device__ __forceinline__ static void image_fast(double* acc, double rx, double ry, const double* w,
                                                    const NearArgs& a) {
    const double X = a.beta2 * fma(rx, rx, ry * ry);
    const pwk::K01 k = pwk::k01_asym<LOWP, true, FAR, COARSE>(X);
    acc[0] = fma(w[0], k.k0, acc[0]);
    const double g = w[0] * k.k1_over_x;
    acc[1] = fma(g, rx, acc[1]);
    acc[2] = fma(g, ry, acc[2]);
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs& a, double* out) {
    out[0] = acc[0] * (1.0 / (2.0 * pwk::kPi));
    const double gs = -a.beta2 / (2.0 * pwk::kPi);
    out[1] = acc[1] * gs;
    out[2] = acc[2] * gs;
  }
};

// Stokeslet -(1/4pi)(log|r| I - r r^T/|r|^2) f  (kernels.cpp:115-119), plus the
// optional pressurelet r.f/(2 pi r^2) (kernels.cpp:139-143).
template <bool PRESSURE, bool LOWP>
struct Stokes {
  static constexpr int NW = 2, NACC = PRESSURE ? 5 : 4, NOUT = PRESSURE ? 3 : 2;
  using Consts = pwk::LogK<LOWP>;
  __device__ __forceinline__ static Consts consts() { return pwk::log_consts<LOWP>(); }
  template <int NXI, int NROW>
  __device__ __forceinline__ static void pair(double* acc, double dx, double dy, const double* w,
                                              const NearArgs& a, int& flag, const Consts& C) {
    double P = 1.0;
    double ax = 0.0, ay = 0.0, pr = 0.0;
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
      const double ry2 = ry * ry;
      const double fy_ry = w[1] * ry;
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        const double r2 = fma(rx, rx, ry2);
        P *= r2;
        const double t = fma(w[0], rx, fy_ry) * pwk::rcp_tier<LOWP>(r2);
        ax = fma(rx, t, ax);
        ay = fma(ry, t, ay);
        if (PRESSURE) pr += t;
      }
    }
    int bad = 0;
    const double L = pwk::log_pos_k<LOWP>(P, C, bad);
    if (!bad) {
      acc[0] = fma(L, w[0], acc[0]);
      acc[1] = fma(L, w[1], acc[1]);
      acc[2] += ax;
      acc[3] += ay;
      if (PRESSURE) acc[4] += pr;
      return;
    }
    // slow path: exact per-image semantics (rare: coincident or extreme pairs)
#pragma unroll 1
    for (int n = 0; n < NROW; ++n)
#pragma unroll 1
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        const double ry = row_dy<NXI, NROW>(dy, a, n);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        const double r2 = fma(rx, rx, ry * ry);
        const double L = pwk::log_r2_safe(rx, ry);
        const double t = fma(w[0], rx, w[1] * ry) / r2;
        acc[0] = fma(L, w[0], acc[0]);
        acc[1] = fma(L, w[1], acc[1]);
        acc[2] = fma(rx, t, acc[2]);
        acc[3] = fma(ry, t, acc[3]);
        if (PRESSURE) acc[4] += t;
      }
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    const double c = -1.0 / (4.0 * pwk::kPi);
    out[0] = c * fma(0.5, acc[0], -acc[2]);
    out[1] = c * fma(0.5, acc[1], -acc[3]);
    if (PRESSURE) out[2] = acc[4] * (1.0 / (2.0 * pwk::kPi));
  }
};

// Screened Stokeslet (kernels.cpp:120-130) through g1/g2 (kernels.cpp:36-68).
template <bool PRESSURE>
struct ModStokes {
  static constexpr int NW = 2, NACC = PRESSURE ? 3 : 2, NOUT = PRESSURE ? 3 : 2;
  template <int NXI, int NROW>
  __device__ __forceinline__ static void pair(double* acc, double dx, double dy, const double* w,
                                              const NearArgs& a, int& flag) {
#pragma unroll 1
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
#pragma unroll 1
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        const double r2 = fma(rx, rx, ry * ry);
        const double inv = 1.0 / r2;
        const pwk::G12 g = pwk::mod_stokes_g12(a.beta * sqrt(r2));
        const double c = inv * a.ms_scale;  // 1/(2 pi beta^2 r^2)
        const double xh2 = rx * rx * inv, yh2 = ry * ry * inv, xy = rx * ry * inv;
        const double g11 = c * (g.g2 * yh2 + g.g1 * xh2);
        const double g22 = c * (g.g2 * xh2 + g.g1 * yh2);
        const double g12 = -c * xy * (g.g2 - g.g1);
        acc[0] += g11 * w[0] + g12 * w[1];
        acc[1] += g12 * w[0] + g22 * w[1];
        if (PRESSURE) acc[2] += fma(rx, w[0], ry * w[1]) * inv;
      }
    }
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0];
    out[1] = acc[1];
    if (PRESSURE) out[2] = acc[2] * (1.0 / (2.0 * pwk::kPi));
  }
};

// Stresslet double layer -(1/pi) r r^T (r.n) f / |r|^4 (kernels.cpp:145-151).
struct Stresslet {
  static constexpr int NW = 4, NACC = 2, NOUT = 2;
  template <int NXI, int NROW>
  __device__ __forceinline__ static void pair(double* acc, double dx, double dy, const double* w,
                                              const NearArgs& a, int& flag) {
#pragma unroll
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
#pragma unroll
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        const double r2 = fma(rx, rx, ry * ry);
        const double inv = pwk::rcp(r2);
        const double c = fma(rx, w[2], ry * w[3]) * fma(rx, w[0], ry * w[1]) * inv * inv;
        acc[0] = fma(c, rx, acc[0]);
        acc[1] = fma(c, ry, acc[1]);
      }
    }
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0] * (-1.0 / pwk::kPi);
    out[1] = acc[1] * (-1.0 / pwk::kPi);
  }
};

// Multipole sources (kernels.cpp:153-162): Poisson 1/z^l, ModHelmholtz
// K_l(beta r) (z/r)^l, complex strengths.
struct Multipole {
  static constexpr int NW = 2, NACC = 2, NOUT = 2;
  template <int NXI, int NROW>
  __device__ __forceinline__ static void pair(double* acc, double dx, double dy, const double* w,
                                              const NearArgs& a, int& flag) {
#pragma unroll 1
    for (int n = 0; n < NROW; ++n) {
      const double ry = row_dy<NXI, NROW>(dy, a, n);
#pragma unroll 1
      for (int m = 0; m < NXI; ++m) {
        const double rx = img_dx<NXI, NROW>(dx, a, n, m);
        if (rx == 0.0 && ry == 0.0) {
          if (n * NXI + m != a.id_img) flag = 1;
          continue;
        }
        double vr, vi;
        if (a.screened) {
          const double r2 = fma(rx, rx, ry * ry);
          const double rr = sqrt(r2);
          const double x = a.beta * rr;
          double kl;
          if (x > 700.0) {
            kl = 0.0;
          } else {
            const pwk::K01 k = pwk::k01_of_sq(x * x);
            double km = k.k0, kc = k.k1_over_x * x;
            for (int l = 1; l < a.order; ++l) {
              const double kn = km + (2.0 * l / x) * kc;
              km = kc;
              kc = kn;
            }
            kl = kc;
          }
          // (z / r)^l
          const double ux = rx / rr, uy = ry / rr;
          double pr = 1.0, pi = 0.0;
          for (int l = 0; l < a.order; ++l) {
            const double t = pr * ux - pi * uy;
            pi = pr * uy + pi * ux;
            pr = t;
          }
          vr = kl * pr;
          vi = kl * pi;
        } else {
          // 1 / z^l: z^l by repeated multiplication, then complex reciprocal
          double pr = 1.0, pi = 0.0;
          for (int l = 0; l < a.order; ++l) {
            const double t = pr * rx - pi * ry;
            pi = pr * ry + pi * rx;
            pr = t;
          }
          const double d = pr * pr + pi * pi;
          vr = pr / d;
          vi = -pi / d;
        }
        acc[0] += vr * w[0] - vi * w[1];
        acc[1] += vr * w[1] + vi * w[0];
      }
    }
  }
  __device__ __forceinline__ static void finish(const double* acc, const NearArgs&, double* out) {
    out[0] = acc[0];
    out[1] = acc[1];
  }
};

// ---------------------------------------------------------------- the tile kernel
// Functors with per-thread constants (KER::Consts, e.g. the log coefficients) get them
// built once per thread and passed to every pair.
struct NoConsts {};
template <class K, class = void>
struct HasConsts : std::false_type {
  using type = NoConsts;
  __device__ __forceinline__ static type make() { return {}; }
};
template <class K>
struct HasConsts<K, std::void_t<typename K::Consts>> : std::true_type {
  using type = typename K::Consts;
  __device__ __forceinline__ static type make() { return K::consts(); }
};

template <class K, class = void>
struct ImageOuter : std::false_type {};
template <class K>
struct ImageOuter<K, std::enable_if_t<K::IMAGE_OUTER>> : std::true_type {};

template <class K, class = void>
struct UsesExpTab : std::false_type {};
template <class K>
struct UsesExpTab<K, std::enable_if_t<K::EXP_TAB>> : std::true_type {};

template <class KER, int NXI, int NROW, int TPT>
__global__ void __launch_bounds__(kThreads) near_tile_kernel(const __grid_constant__ NearArgs a) {
  __shared__ double s_x[kTile];
  __shared__ double s_y[kTile];
  __shared__ double s_w[KER::NW][kTile];

  const size_t block_t0 = static_cast<size_t>(blockIdx.x) * (kThreads * TPT);
  double tx[TPT], ty[TPT], acc[TPT][KER::NACC];
  bool live[TPT];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const size_t l = block_t0 + threadIdx.x + k * kThreads;
    live[k] = l < a.nt;
    const double2 t = live[k] ? a.tgt[l] : make_double2(0.0, 0.0);
    tx[k] = t.x;
    ty[k] = t.y;
#pragma unroll
    for (int c = 0; c < KER::NACC; ++c) acc[k][c] = 0.0;
  }
  int flag = 0;
  const typename HasConsts<KER>::type C = HasConsts<KER>::make();
  if constexpr (UsesExpTab<KER>::value) pwk::exp_tab_fill();  // visible after the tile loop's first __syncthreads
  // screened kernels: bounding boxes of the block's targets and of each source tile give
  // per-image masks and regimes (binned inputs make both compact; near_sym_impl.cuh)
  constexpr bool kBoxes = ImageOuter<KER>::value;
  constexpr int kWarpsT = kThreads / 32;
  __shared__ double s_tbox[kBoxes ? kWarpsT : 1][4], s_sbox[kBoxes ? kWarpsT : 1][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    warp_box_store(b[0], b[1], b[2], b[3], lane, s_tbox[warp]);  // read after the loop's syncs
  }

  const size_t j_begin = static_cast<size_t>(blockIdx.y) * a.src_per_split;
  size_t j_end = j_begin + a.src_per_split;
  if (j_end > a.ns) j_end = a.ns;

  for (size_t j0 = j_begin; j0 < j_end; j0 += kTile) {
    const int tn = static_cast<int>((j_end - j0) < kTile ? (j_end - j0) : kTile);
    __syncthreads();
    double sb[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    for (int i = threadIdx.x; i < tn; i += kThreads) {
      const double2 p = a.src[j0 + i];
      s_x[i] = p.x;
      s_y[i] = p.y;
      if (kBoxes) {
        sb[0] = fmin(sb[0], p.x);
        sb[1] = fmin(sb[1], -p.x);
        sb[2] = fmin(sb[2], p.y);
        sb[3] = fmin(sb[3], -p.y);
      }
      if (KER::NW == 1) {
        s_w[0][i] = a.q[j0 + i];
      } else {
        const double2 v = a.vec[j0 + i];
        s_w[0][i] = v.x;
        s_w[1 % KER::NW][i] = v.y;
        if (KER::NW == 4) {
          const double2 nn = a.nrm[j0 + i];
          s_w[2 % KER::NW][i] = nn.x;
          s_w[3 % KER::NW][i] = nn.y;
        }
      }
    }
    if constexpr (kBoxes) warp_box_store(sb[0], sb[1], sb[2], sb[3], lane, s_sbox[warp]);
    __syncthreads();
    if constexpr (ImageOuter<KER>::value) {
      // screened kernels: image-outer order (loop-invariant shift, one K0 per inner
      // iteration, small code; near_sym_impl.cuh does the same on its off-diagonal tiles);
      // an image whose box range lies beyond the cut-off is skipped, one whose range lies in
      // one asymptotic regime runs branch-free (same arithmetic as the per-pair dispatch)
      double tb[4], sbx[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tb[c] = fmin(fmin(s_tbox[0][c], s_tbox[1][c]), fmin(s_tbox[2][c], s_tbox[3][c]));
        sbx[c] = fmin(fmin(s_sbox[0][c], s_sbox[1][c]), fmin(s_sbox[2][c], s_sbox[3][c]));
      }
#pragma unroll 1
      for (int img = 0; img < NXI * NROW; ++img) {
        const double shx = a.shx[img], shy = a.shy[img / NXI];
        const bool ident = img == a.id_img;
        double lo, hi;
        image_xrange(tb, sbx, shx, shy, a.beta2, lo, hi);
        if (a.cull && lo * 0.9999 >= a.xcut2) continue;  // block-uniform
        const int regime = a.cull ? pwk::regime_of(lo, hi, a.xcut2) : 0;
        auto sweep = [&](auto reg) {
          constexpr int R = decltype(reg)::value;
          // regime sweeps: shifted targets once per image, (t - shift) - s (no coincidence is
          // possible there); the per-pair dispatch keeps the reference's (t - s) - shift
          // (apply.cpp:534), whose exact zeros decide CoincidentSourceTarget
          double txs[TPT], tys[TPT];
#pragma unroll
          for (int k = 0; k < TPT; ++k) {
            txs[k] = tx[k] - shx;
            tys[k] = ty[k] - shy;
          }
          constexpr int kU = R == 0 ? PWB_MH_GEN_UNROLL : kMhSrcUnroll;  // the per-pair dispatch is branchy: less unrolled
#pragma unroll kU
          for (int i = 0; i < tn; ++i) {
            const double sx = s_x[i], sy = s_y[i];
            double w[KER::NW];
#pragma unroll
            for (int c = 0; c < KER::NW; ++c) w[c] = s_w[c][i];
#pragma unroll
            for (int k = 0; k < TPT; ++k) {
              const double rx = R == 0 ? (tx[k] - sx) - shx : txs[k] - sx;
              const double ry = R == 0 ? (ty[k] - sy) - shy : tys[k] - sy;
              if constexpr (R == 0)
                KER::image(acc[k], rx, ry, w, ident, a, flag);
              else
                KER::template image_fast<R == 2>(acc[k], rx, ry, w, a);
            }
          }
        };
        if (regime == 2)
          sweep(std::integral_constant<int, 2>{});
        else if (regime == 1 && PWB_MH_NEAR_SWEEP)
          sweep(std::integral_constant<int, 1>{});
        else
          sweep(std::integral_constant<int, 0>{});
      }
    } else {
#pragma unroll 2
      for (int i = 0; i < tn; ++i) {
        const double sx = s_x[i], sy = s_y[i];
        double w[KER::NW];
#pragma unroll
        for (int c = 0; c < KER::NW; ++c) w[c] = s_w[c][i];
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          // (t - s) - shift, the reference's association (apply.cpp:534)
          if constexpr (HasConsts<KER>::value)
            KER::template pair<NXI, NROW>(acc[k], tx[k] - sx, ty[k] - sy, w, a, flag, C);
          else
            KER::template pair<NXI, NROW>(acc[k], tx[k] - sx, ty[k] - sy, w, a, flag);
        }
      }
    }
  }

  if (flag) atomicOr(a.flag, 1);
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    if (!live[k]) continue;
    const size_t l = block_t0 + threadIdx.x + k * kThreads;
    double o[KER::NOUT];
    KER::finish(acc[k], a, o);
    if (a.splits == 1) {
      const size_t row = a.out_row ? static_cast<size_t>(a.out_row[l]) : l;
#pragma unroll
      for (int c = 0; c < KER::NOUT; ++c) {
        double* dst = c < a.nout0 ? a.out0 + row * a.nout0 + c : a.out1 + row * a.nout1 + (c - a.nout0);
        *dst += o[c];
      }
    } else {
      double* part = a.partial + (static_cast<size_t>(blockIdx.y) * a.nt + l) * KER::NOUT;
#pragma unroll
      for (int c = 0; c < KER::NOUT; ++c) part[c] = o[c];
    }
  }
}

// out += sum_split partial[split] in fixed split order.
__global__ void near_reduce_kernel(const double* partial, int splits, size_t nt, int nout, double* out0, int nout0,
                                   double* out1, int nout1, const int* out_row) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= nt * nout) return;
  const size_t l = idx / nout;
  const int c = static_cast<int>(idx % nout);
  double s = 0.0;
  for (int sp = 0; sp < splits; ++sp) s += partial[static_cast<size_t>(sp) * nt * nout + idx];
  const size_t row = out_row ? static_cast<size_t>(out_row[l]) : l;
  double* dst = c < nout0 ? out0 + row * nout0 + c : out1 + row * nout1 + (c - nout0);
  *dst += s;
}

// The same with one warp per output (small target counts with many splits: c1 sums 63
// partials per output); lanes stride over the splits, fixed-order xor-shuffle tree.
__global__ void near_reduce_warp_kernel(const double* partial, int splits, size_t nt, int nout, double* out0,
                                        int nout0, double* out1, int nout1, const int* out_row) {
  const size_t idx = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= nt * nout) return;
  double s = 0.0;
  for (int sp = lane; sp < splits; sp += 32) s += partial[static_cast<size_t>(sp) * nt * nout + idx];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane != 0) return;
  const size_t l = idx / nout;
  const int c = static_cast<int>(idx % nout);
  const size_t row = out_row ? static_cast<size_t>(out_row[l]) : l;
  double* dst = c < nout0 ? out0 + row * nout0 + c : out1 + row * nout1 + (c - nout0);
  *dst += s;
}

template <class KER, int NXI, int NROW, int TPT>
void launch_shape(const NearArgs& a0, cudaStream_t st, double* partial_ws, int sm_count) {
  NearArgs a = a0;
  const size_t per_block = static_cast<size_t>(kThreads) * TPT;
  const unsigned bx = static_cast<unsigned>((a.nt + per_block - 1) / per_block);
  // Source splits: the grid should cover >= 8 waves of resident blocks, with the
  // split count chosen so the last wave is as full as possible (ncu r1, c2: 782
  // blocks on 592 slots left the second wave 32 % occupied, fp64 pipe 61 %).
  // Each split keeps >= 16 sources (c1: 1000 x 1000 runs 4 target blocks x 63 splits).
  // per instantiation: blocks per SM at this kernel's registers/smem (thread-safe static
  // init; the value depends only on the kernel and the sm_100a target, not the device)
  static const int resident = [] {
    int r = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, near_tile_kernel<KER, NXI, NROW, TPT>, kThreads, 0),
               "occupancy");
    return r > 0 ? r : 1;
  }();
  const size_t slots = static_cast<size_t>(sm_count) * resident;
  int splits = 1;
  if (partial_ws != nullptr && bx < 8 * slots) {
    const size_t max_by_src = (a.ns + 15) / 16;
    const int hi = static_cast<int>(std::min<size_t>({static_cast<size_t>(kMaxSplits), max_by_src,
                                                      (8 * slots + bx - 1) / bx + 8}));
    const int lo = std::max(1, std::min(hi, static_cast<int>((8 * slots + bx - 1) / bx)));
    double best = 1e300;
    for (int sp = lo; sp <= hi; ++sp) {  // fewest idle slot-waves per unit of work
      const double blocks = static_cast<double>(bx) * sp;
      const double waste = std::ceil(blocks / slots) * slots / blocks;
      if (waste < best - 1e-9) {
        best = waste;
        splits = sp;
      }
    }
    if (hi < lo) splits = std::max(1, hi);
  }
  a.splits = splits;
  a.src_per_split = (a.ns + splits - 1) / splits;
  a.src_per_split = ((a.src_per_split + 7) / 8) * 8;
  a.partial = partial_ws;
  dim3 grid(bx, splits);
  // with splits the tile only writes partials: it may run on the branch stream, joined here
  cudaStream_t ts = (a.tile_stream && splits > 1) ? static_cast<cudaStream_t>(a.tile_stream) : st;
  near_tile_kernel<KER, NXI, NROW, TPT><<<grid, kThreads, 0, ts>>>(a);
  count_launches(1);
  if (a.tile_stream) {  // always join the branch (it may have been forked with nothing on it)
    auto done = static_cast<cudaEvent_t>(a.tile_done);
    cuda_check(cudaEventRecord(done, static_cast<cudaStream_t>(a.tile_stream)), "tile join");
    cuda_check(cudaStreamWaitEvent(st, done, 0), "tile join wait");
  }
  if (splits > 1) {
    const size_t n = a.nt * KER::NOUT;
    if (n < 65536 && splits >= 8)
      near_reduce_warp_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, st>>>(
          partial_ws, splits, a.nt, KER::NOUT, a.out0, a.nout0, a.out1, a.nout1, a.out_row);
    else
      near_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(partial_ws, splits, a.nt, KER::NOUT,
                                                                                 a.out0, a.nout0, a.out1, a.nout1,
                                                                                 a.out_row);
    count_launches(1);
  }
}

template <class KER, int TPT>
void dispatch_images(const NearArgs& a, cudaStream_t st, double* ws, int sms) {
  if (a.nxi == 1 && a.nrow == 1) return launch_shape<KER, 1, 1, TPT>(a, st, ws, sms);
  if (a.nxi == 3 && a.nrow == 1) return launch_shape<KER, 3, 1, TPT>(a, st, ws, sms);
  if (a.nxi == 3 && a.nrow == 3) return launch_shape<KER, 3, 3, TPT>(a, st, ws, sms);
  if (a.nxi == 5 && a.nrow == 3) return launch_shape<KER, 5, 3, TPT>(a, st, ws, sms);
  if (a.nxi == 7 && a.nrow == 3) return launch_shape<KER, 7, 3, TPT>(a, st, ws, sms);
  throw_internal("near field: unsupported image layout");
}

}  // namespace

size_t near_outputs(NearKind kind) {
  switch (kind) {
    case NearKind::Laplace:
    case NearKind::ModHelm: return 1;
    case NearKind::ModHelmGrad: return 3;
    case NearKind::Stokes:
    case NearKind::ModStokes:
    case NearKind::Stresslet:
    case NearKind::Multipole: return 2;
    case NearKind::StokesP:
    case NearKind::ModStokesP: return 3;
  }
  return 1;
}

void launch_near(NearKind kind, const NearArgs& a, cudaStream_t st, double* partial_ws, int sm_count) {
  if (a.nt == 0 || a.ns == 0) return;
  switch (kind) {
    case NearKind::Laplace:
      return a.lowp ? dispatch_images<Laplace<true>, 2>(a, st, partial_ws, sm_count)
                    : dispatch_images<Laplace<false>, 2>(a, st, partial_ws, sm_count);
    // precision tier (pw_math.cuh k01_tile): reduced when eps allows it
    case NearKind::ModHelm:
      if (a.lowp == 2) return dispatch_images<ModHelm<true, true>, PWB_MH_TPT>(a, st, partial_ws, sm_count);
      return a.lowp ? dispatch_images<ModHelm<true>, PWB_MH_TPT>(a, st, partial_ws, sm_count)
                    : dispatch_images<ModHelm<false>, PWB_MH_TPT>(a, st, partial_ws, sm_count);
    case NearKind::ModHelmGrad:
      if (a.lowp == 2) return dispatch_images<ModHelmGrad<true, true>, PWB_MH_TPT>(a, st, partial_ws, sm_count);
      return a.lowp ? dispatch_images<ModHelmGrad<true>, PWB_MH_TPT>(a, st, partial_ws, sm_count)
                    : dispatch_images<ModHelmGrad<false>, PWB_MH_TPT>(a, st, partial_ws, sm_count);
    case NearKind::Stokes:
      return a.lowp ? dispatch_images<Stokes<false, true>, 1>(a, st, partial_ws, sm_count)
                    : dispatch_images<Stokes<false, false>, 1>(a, st, partial_ws, sm_count);
    case NearKind::StokesP:
      return a.lowp ? dispatch_images<Stokes<true, true>, 1>(a, st, partial_ws, sm_count)
                    : dispatch_images<Stokes<true, false>, 1>(a, st, partial_ws, sm_count);
    case NearKind::ModStokes: return dispatch_images<ModStokes<false>, 1>(a, st, partial_ws, sm_count);
    case NearKind::ModStokesP: return dispatch_images<ModStokes<true>, 1>(a, st, partial_ws, sm_count);
    case NearKind::Stresslet: return dispatch_images<Stresslet, 1>(a, st, partial_ws, sm_count);
    case NearKind::Multipole: return dispatch_images<Multipole, 1>(a, st, partial_ws, sm_count);
  }
}

}  // namespace pwb
