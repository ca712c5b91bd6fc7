// Direct plane-wave contractions of the far field: S2PW source sums, the
// per-mode diagonal/block finalisation, and PW2T target evaluation.
//
// Replaces add_scalar_modes_direct / add_block_direct / add_pressure_direct /
// add_stresslet_direct and the m0 rank-one terms
// (/root/reference/proj/src/apply.cpp:32-192) with mode factors
//   source  S_j(r) = e^{decay_s (w_j - shift_s)} e^{-i phase p_j}   (apply.cpp:32-34)
//   target  T_l(r) = e^{decay_t (w_l - shift_t)} e^{+i phase p_l}   (apply.cpp:36-38)
// evaluated on the fly (no r x N matrix is ever materialised). The S2PW sums
// are reduced warp-shuffle -> shared memory -> per-chunk partials -> fixed-order
// chunk sum, so results are run-to-run deterministic and the raw sums are
// linear in the sources (the multi-GPU allreduce operand).
#include <cuda_runtime.h>

#include <type_traits>

#include "pw_engine.cuh"

namespace pwb {
namespace {

constexpr int kS2pwThreads = 128;

// Per-source raw strengths -> K real weights for a mode of axis `ax`.
template <WeightSet WS>
struct Weights;

template <>
struct Weights<WeightSet::Charge> {
  static constexpr int K = 1;
  __device__ static void load(const S2pwArgs& a, size_t j, double* raw) { raw[0] = a.q[j]; }
  __device__ static void make(const double* raw, double, double* w) { w[0] = raw[0]; }
};
template <>
struct Weights<WeightSet::Coef> {
  static constexpr int K = 2;
  __device__ static void load(const S2pwArgs& a, size_t j, double* raw) {
    const double2 v = a.vec[j];
    raw[0] = v.x;
    raw[1] = v.y;
  }
  __device__ static void make(const double* raw, double, double* w) {
    w[0] = raw[0];
    w[1] = raw[1];
  }
};
template <>
struct Weights<WeightSet::Force> : Weights<WeightSet::Coef> {};
template <>
struct Weights<WeightSet::ForceW> {
  static constexpr int K = 4;
  __device__ static void load(const S2pwArgs& a, size_t j, double* raw) {
    const double2 v = a.vec[j];
    raw[0] = v.x;
    raw[1] = v.y;
  }
  __device__ static void make(const double* raw, double wc, double* w) {
    w[0] = raw[0];
    w[1] = raw[1];
    w[2] = wc * raw[0];  // s2 = sum w_j S f_j (apply.cpp:92)
    w[3] = wc * raw[1];
  }
};
template <>
struct Weights<WeightSet::DoubleLayer> {
  static constexpr int K = 8;
  __device__ static void load(const S2pwArgs& a, size_t j, double* raw) {
    const double2 v = a.vec[j];
    const double2 n = a.nrm[j];
    raw[0] = v.x;
    raw[1] = v.y;
    raw[2] = n.x;
    raw[3] = n.y;
  }
  __device__ static void make(const double* raw, double wc, double* w) {  // apply.cpp:160-164
    w[0] = raw[2] * raw[0];
    w[1] = raw[2] * raw[1];
    w[2] = raw[3] * raw[0];
    w[3] = raw[3] * raw[1];
    const double n1w = raw[2] * wc, n2w = raw[3] * wc;
    w[4] = n1w * raw[0];
    w[5] = n1w * raw[1];
    w[6] = n2w * raw[0];
    w[7] = n2w * raw[1];
  }
};

template <WeightSet WS, int MT>
__global__ void __launch_bounds__(kS2pwThreads) s2pw_kernel(const __grid_constant__ S2pwArgs a) {
  using W = Weights<WS>;
  constexpr int K = W::K;
  constexpr int NV = MT * K * 2;
  const int r0 = blockIdx.x * MT;
  double ph[MT], ds[MT], ss[MT];
  int ax[MT];
  bool alive[MT];
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int r = r0 + t;
    alive[t] = r < a.modes.count;
    const int rr = alive[t] ? r : 0;
    ph[t] = a.modes.phase[rr];
    ds[t] = a.modes.decay_s[rr];
    ss[t] = a.modes.shift_s[rr];
    ax[t] = a.modes.axis[rr];
  }
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;

  const size_t j0 = static_cast<size_t>(blockIdx.y) * a.per_chunk;
  size_t j1 = j0 + a.per_chunk;
  if (j1 > a.ns) j1 = a.ns;
  for (size_t j = j0 + threadIdx.x; j < j1; j += kS2pwThreads) {
    const double2 p = a.src[j];
    double raw[4];
    W::load(a, j, raw);
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const double wc = ax[t] ? p.x : p.y;  // decay coordinate (apply.cpp:29)
      const double pc = ax[t] ? p.y : p.x;  // oscillation coordinate (apply.cpp:30)
      const double mag = exp(ds[t] * (wc - ss[t]));
      double sn, cs;
      sincos(ph[t] * pc, &sn, &cs);
      const double sre = mag * cs, sim = -mag * sn;
      double w[K];
      W::make(raw, wc, w);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        acc[(t * K + k) * 2] = fma(sre, w[k], acc[(t * K + k) * 2]);
        acc[(t * K + k) * 2 + 1] = fma(sim, w[k], acc[(t * K + k) * 2 + 1]);
      }
    }
  }

  __shared__ double red[kS2pwThreads / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double x = acc[v];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if (lane == 0) red[warp][v] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int wv = 0; wv < kS2pwThreads / 32; ++wv) s += red[wv][threadIdx.x];
    const int t = threadIdx.x / (2 * K);
    if (r0 + t < a.modes.count) {
      const size_t base = (static_cast<size_t>(blockIdx.y) * a.modes.count + r0) * K * 2;
      a.partial[base + threadIdx.x] = s;
    }
  }
}

template <WeightSet WS>
void s2pw_dispatch(const S2pwArgs& a, cudaStream_t st) {
  constexpr int K = Weights<WS>::K;
  constexpr int MT = K >= 8 ? 1 : 8 / K;
  if (a.narrow) {  // c1: 1344 + 32 blocks of 128 threads, 8 sources per thread, no chunk sum
    s2pw_kernel<WS, 1><<<dim3(a.modes.count, a.chunks), kS2pwThreads, 0, st>>>(a);
  } else {
    dim3 grid((a.modes.count + MT - 1) / MT, a.chunks);
    s2pw_kernel<WS, MT><<<grid, kS2pwThreads, 0, st>>>(a);
  }
  count_launches(1);
}

__global__ void chunk_sum_kernel(const double* partial, int chunks, size_t len, double* raw) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= len) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += partial[static_cast<size_t>(c) * len + i];
  raw[i] = s;
}

// ---------------------------------------------------------------- complex helpers
struct C2 {
  double re, im;
};
__device__ __forceinline__ C2 ld(const double* p) { return {p[0], p[1]}; }
__device__ __forceinline__ C2 cmul(C2 a, C2 b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ C2 cadd(C2 a, C2 b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ C2 csub(C2 a, C2 b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ void st(double* p, C2 v) {
  p[0] = v.re;
  p[1] = v.im;
}
// Mat2c (8 doubles, row-major) times Vec2c
__device__ __forceinline__ void mat_vec(const double* m, C2 x, C2 y, C2* ox, C2* oy) {
  *ox = cadd(cmul(ld(m), x), cmul(ld(m + 2), y));
  *oy = cadd(cmul(ld(m + 4), x), cmul(ld(m + 6), y));
}

__global__ void prep_kernel(const __grid_constant__ PrepArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.count) return;
  const double* raw = a.raw + static_cast<size_t>(r) * a.k * 2;
  switch (a.kind) {
    case FamilyKind::Scalar: {  // apply.cpp:57 srcsum = diag * s
      C2 s = ld(raw);
      if (a.k == 2) {  // complex strengths: s0 + i s1
        const C2 s1 = ld(raw + 2);
        s = {s.re - s1.im, s.im + s1.re};
      }
      st(a.A + 2 * r, cmul(ld(a.t0 + 2 * r), s));
      break;
    }
    case FamilyKind::Block: {  // apply.cpp:101-104
      const C2 s1x = ld(raw), s1y = ld(raw + 2);
      C2 ax, ay;
      mat_vec(a.t0 + 8 * r, s1x, s1y, &ax, &ay);
      if (a.three_term[r]) {
        const C2 s2x = ld(raw + 4), s2y = ld(raw + 6);
        C2 bx, by, cx, cy;
        mat_vec(a.t1 + 8 * r, s2x, s2y, &bx, &by);
        mat_vec(a.t1 + 8 * r, s1x, s1y, &cx, &cy);
        ax = cadd(ax, bx);
        ay = cadd(ay, by);
        st(a.B + 4 * r, {-cx.re, -cx.im});
        st(a.B + 4 * r + 2, {-cy.re, -cy.im});
      } else {
        st(a.B + 4 * r, {0.0, 0.0});
        st(a.B + 4 * r + 2, {0.0, 0.0});
      }
      st(a.A + 4 * r, ax);
      st(a.A + 4 * r + 2, ay);
      break;
    }
    case FamilyKind::Pressure: {  // apply.cpp:128-131
      const double* row = a.t1 + 4 * r;
      const C2 s = cadd(cmul(ld(row), ld(raw)), cmul(ld(row + 2), ld(raw + 2)));
      st(a.A + 2 * r, cmul(ld(a.t0 + 2 * r), s));
      break;
    }
    case FamilyKind::Stresslet: {  // apply.cpp:166-170
      const C2 v1x = ld(raw), v1y = ld(raw + 2), v2x = ld(raw + 4), v2y = ld(raw + 6);
      const C2 v3x = ld(raw + 8), v3y = ld(raw + 10), v4x = ld(raw + 12), v4y = ld(raw + 14);
      const C2 sa = ld(a.t3 + 2 * r), sb = ld(a.t4 + 2 * r), off = ld(a.t5 + 2 * r);
      const C2 ux = cadd(cmul(sa, v1x), cmul(sb, v2x)), uy = cadd(cmul(sa, v1y), cmul(sb, v2y));
      C2 q1x, q1y;
      mat_vec(a.t2 + 8 * r, ux, uy, &q1x, &q1y);
      const C2 wx = cadd(cmul(sa, v3x), cmul(sb, v4x)), wy = cadd(cmul(sa, v3y), cmul(sb, v4y));
      C2 mx, my, a1x, a1y, a2x, a2y;
      mat_vec(a.t2 + 8 * r, wx, wy, &mx, &my);
      mat_vec(a.t0 + 8 * r, v1x, v1y, &a1x, &a1y);
      mat_vec(a.t1 + 8 * r, v2x, v2y, &a2x, &a2y);
      const C2 q0x = csub(cadd(cadd(a1x, a2x), cmul(off, q1x)), mx);
      const C2 q0y = csub(cadd(cadd(a1y, a2y), cmul(off, q1y)), my);
      st(a.A + 4 * r, q0x);
      st(a.A + 4 * r + 2, q0y);
      st(a.B + 4 * r, q1x);
      st(a.B + 4 * r + 2, q1y);
      break;
    }
  }
}

// ---------------------------------------------------------------- PW2T
constexpr int kPw2tThreads = 128;
constexpr int kModeTile = 128;

template <int KO, bool HASB, bool GRAD>
__global__ void __launch_bounds__(kPw2tThreads) pw2t_kernel(const __grid_constant__ Pw2tArgs a) {
  __shared__ double s_ph[kModeTile], s_dt[kModeTile], s_st[kModeTile];
  __shared__ int s_ax[kModeTile];
  __shared__ double s_A[kModeTile][KO * 2];
  __shared__ double s_B[HASB ? kModeTile : 1][KO * 2];

  const size_t l = static_cast<size_t>(blockIdx.x) * kPw2tThreads + threadIdx.x;
  const bool live = l < a.nt;
  const double2 t = live ? a.tgt[l] : make_double2(0.0, 0.0);
  double acc[KO * 2];
#pragma unroll
  for (int v = 0; v < KO * 2; ++v) acc[v] = 0.0;
  double gx_re = 0.0, gx_im = 0.0, gy_re = 0.0, gy_im = 0.0;

  for (int r0 = 0; r0 < a.modes.count; r0 += kModeTile) {
    const int tn = min(kModeTile, a.modes.count - r0);
    __syncthreads();
    for (int i = threadIdx.x; i < tn; i += kPw2tThreads) {
      s_ph[i] = a.modes.phase[r0 + i];
      s_dt[i] = a.modes.decay_t[r0 + i];
      s_st[i] = a.modes.shift_t[r0 + i];
      s_ax[i] = a.modes.axis[r0 + i];
#pragma unroll
      for (int v = 0; v < KO * 2; ++v) {
        s_A[i][v] = a.A[static_cast<size_t>(r0 + i) * KO * 2 + v];
        if (HASB) s_B[i][v] = a.B[static_cast<size_t>(r0 + i) * KO * 2 + v];
      }
    }
    __syncthreads();
    for (int i = 0; i < tn; ++i) {
      const int ax = s_ax[i];
      const double wc = ax ? t.x : t.y;
      const double pc = ax ? t.y : t.x;
      const double mag = exp(s_dt[i] * (wc - s_st[i]));
      double sn, cs;
      sincos(s_ph[i] * pc, &sn, &cs);
      const double tre = mag * cs, tim = mag * sn;
#pragma unroll
      for (int k = 0; k < KO; ++k) {
        double cre = s_A[i][2 * k], cim = s_A[i][2 * k + 1];
        if (HASB) {
          cre = fma(wc, s_B[i][2 * k], cre);
          cim = fma(wc, s_B[i][2 * k + 1], cim);
        }
        acc[2 * k] += tre * cre - tim * cim;
        acc[2 * k + 1] += tre * cim + tim * cre;
      }
      if (GRAD) {
        // d/dx, d/dy of T: vertical (i phase, decay_t), horizontal (decay_t, i phase)
        const double cre = s_A[i][0], cim = s_A[i][1];
        const double pre = tre * cre - tim * cim, pim = tre * cim + tim * cre;
        const double ph = s_ph[i], dt = s_dt[i];
        const double ire = -ph * pim, iim = ph * pre;  // i phase * TC
        const double dre = dt * pre, dim = dt * pim;   // decay_t * TC
        if (ax) {
          gx_re += dre;
          gx_im += dim;
          gy_re += ire;
          gy_im += iim;
        } else {
          gx_re += ire;
          gx_im += iim;
          gy_re += dre;
          gy_im += dim;
        }
      }
    }
  }
  if (!live) return;
  if (a.m0_lin) {  // apply.cpp:68-78 / :108-117: acc += w_l * moment (vertical parts: w = y)
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) acc[v] = fma(t.y, a.m0_lin[v], acc[v]);
    if (GRAD) {
      gy_re += a.m0_lin[0];
      gy_im += a.m0_lin[1];
    }
  }
  if (a.m0_const) {  // apply.cpp:140-146 (pressure constant)
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) acc[v] += a.m0_const[v];
  }
  if (a.out_re) {
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      double* dst = a.out_re + l * KO + k;
      *dst = a.accumulate ? *dst + acc[2 * k] : acc[2 * k];
    }
  }
  if (a.out_cplx) {
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) {
      double* dst = a.out_cplx + l * KO * 2 + v;
      *dst = a.accumulate ? *dst + acc[v] : acc[v];
    }
  }
  if (GRAD && a.out_grad) {
    double* g = a.out_grad + 2 * l;
    g[0] = a.accumulate ? g[0] + gx_re : gx_re;
    g[1] = a.accumulate ? g[1] + gy_re : gy_re;
  }
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ bool inside(double px, double py, double d, double xi, double eta) {
  // cell.cpp:60-70 (closed cell with 1e-12 slack)
  const double x2 = py / eta;
  const double x1 = (px - xi * x2) / d;
  const double lim = 0.5 + 1e-12;
  return fabs(x1) <= lim && fabs(x2) <= lim;
}

constexpr int kRedThreads = 256;

__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const __grid_constant__ ReduceArgs a, double* bm,
                                                             double* bc) {
  double m[kMoments] = {0, 0, 0, 0, 0};
  double c[kChecks] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const size_t stride = static_cast<size_t>(gridDim.x) * kRedThreads;
  for (size_t j = static_cast<size_t>(blockIdx.x) * kRedThreads + threadIdx.x; j < a.ns; j += stride) {
    const double2 p = a.src[j];
    if (!inside(p.x, p.y, a.d, a.xi, a.eta)) c[0] += 1.0;
    if (a.q) {
      const double q = a.q[j];
      m[0] = fma(p.y, q, m[0]);
      c[2] += q;
      c[3] += fabs(q);
    }
    if (a.vec) {
      const double2 f = a.vec[j];
      m[1] = fma(p.y, f.x, m[1]);
      m[2] = fma(p.y, f.y, m[2]);
      c[4] += f.x;
      c[5] += f.y;
      c[6] += hypot(f.x, f.y);
      if (a.nrm) {
        const double2 n = a.nrm[j];
        m[3] += n.y * f.x + n.x * f.y;  // apply.cpp:183-184
        m[4] += n.x * f.x + n.y * f.y;
      }
    }
    if (a.nrm) {
      const double2 n = a.nrm[j];
      if (!(fabs(hypot(n.x, n.y) - 1.0) <= 1e-12)) c[1] += 1.0;
    }
    if (a.coef) {
      const double2 cc = a.coef[j];
      c[7] += cc.x;
      c[8] += cc.y;
      c[9] += hypot(cc.x, cc.y);
    }
  }
  for (size_t l = static_cast<size_t>(blockIdx.x) * kRedThreads + threadIdx.x; l < a.nt; l += stride) {
    const double2 p = a.tgt[l];
    if (!inside(p.x, p.y, a.d, a.xi, a.eta)) c[0] += 1.0;
  }
  __shared__ double red[kRedThreads / 32][kMoments + kChecks];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < kMoments + kChecks; ++v) {
    double x = v < kMoments ? m[v] : c[v - kMoments];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    if (lane == 0) red[warp][v] = x;
  }
  __syncthreads();
  if (threadIdx.x < kMoments + kChecks) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += red[w][threadIdx.x];
    if (threadIdx.x < kMoments)
      bm[blockIdx.x * kMoments + threadIdx.x] = s;
    else
      bc[blockIdx.x * kChecks + threadIdx.x - kMoments] = s;
  }
}

// out[i] = sum_b v[b * n + i]: one warp per value, lanes stride over the blocks, fixed-order
// xor-shuffle tree (deterministic); a serial thread per value took ~20 us at 296 blocks
__global__ void sum_blocks_kernel(const double* v, int blocks, int n, double* out) {
  const int i = static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int b = lane; b < blocks; b += 32) s += v[b * n + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

}  // namespace

void launch_s2pw(WeightSet ws, const S2pwArgs& a, cudaStream_t st) {
  if (a.modes.count == 0) return;
  switch (ws) {
    case WeightSet::Charge: return s2pw_dispatch<WeightSet::Charge>(a, st);
    case WeightSet::Coef: return s2pw_dispatch<WeightSet::Coef>(a, st);
    case WeightSet::Force: return s2pw_dispatch<WeightSet::Force>(a, st);
    case WeightSet::ForceW: return s2pw_dispatch<WeightSet::ForceW>(a, st);
    case WeightSet::DoubleLayer: return s2pw_dispatch<WeightSet::DoubleLayer>(a, st);
  }
}

// Small target counts (c1: 1000 targets = 8 blocks of the kernel above on 148 SMs): G warps
// per target (G = 1: four targets per block; G = 4: one target per block), the group's
// lanes stride over the modes, fixed-order xor-shuffle reduction inside each warp and a
// fixed-order sum over the G warps (deterministic). Same per-(target, mode) arithmetic as
// pw2t_kernel.
template <int KO, bool HASB, bool GRAD, int G>
__global__ void __launch_bounds__(kPw2tThreads) pw2t_warp_kernel(const __grid_constant__ Pw2tArgs a) {
  static_assert(kPw2tThreads % (32 * G) == 0, "whole groups per block");
  constexpr int NV = KO * 2 + 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t l = static_cast<size_t>(blockIdx.x) * (kPw2tThreads / (32 * G)) + warp / G;
  const int gl = (warp % G) * 32 + lane;  // lane inside the target's group
  __shared__ double part[kPw2tThreads / 32][NV];
  const bool live = l < a.nt;
  const double2 t = live ? a.tgt[l] : make_double2(0.0, 0.0);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  for (int r = gl; live && r < a.modes.count; r += 32 * G) {
    const int ax = a.modes.axis[r];
    const double wc = ax ? t.x : t.y;
    const double pc = ax ? t.y : t.x;
    const double ph = a.modes.phase[r], dt = a.modes.decay_t[r];
    const double mag = exp(dt * (wc - a.modes.shift_t[r]));
    double sn, cs;
    sincos(ph * pc, &sn, &cs);
    const double tre = mag * cs, tim = mag * sn;
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      double cre = a.A[static_cast<size_t>(r) * KO * 2 + 2 * k], cim = a.A[static_cast<size_t>(r) * KO * 2 + 2 * k + 1];
      if (HASB) {
        cre = fma(wc, a.B[static_cast<size_t>(r) * KO * 2 + 2 * k], cre);
        cim = fma(wc, a.B[static_cast<size_t>(r) * KO * 2 + 2 * k + 1], cim);
      }
      acc[2 * k] += tre * cre - tim * cim;
      acc[2 * k + 1] += tre * cim + tim * cre;
    }
    if (GRAD) {
      const double cre = a.A[static_cast<size_t>(r) * KO * 2], cim = a.A[static_cast<size_t>(r) * KO * 2 + 1];
      const double pre = tre * cre - tim * cim, pim = tre * cim + tim * cre;
      const double ire = -ph * pim, iim = ph * pre;
      const double dre = dt * pre, dim = dt * pim;
      double* g = acc + KO * 2;  // gx_re, gx_im, gy_re, gy_im
      if (ax) {
        g[0] += dre;
        g[1] += dim;
        g[2] += ire;
        g[3] += iim;
      } else {
        g[0] += ire;
        g[1] += iim;
        g[2] += dre;
        g[3] += dim;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
  if constexpr (G > 1) {
    if (lane == 0)
#pragma unroll
      for (int v = 0; v < NV; ++v) part[warp][v] = acc[v];
    __syncthreads();
    if (warp % G != 0 || lane != 0) return;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double x = part[warp][v];
#pragma unroll
      for (int g = 1; g < G; ++g) x += part[warp + g][v];
      acc[v] = x;
    }
  } else if (lane != 0) {
    return;
  }
  if (!live) return;
  double gx_re = acc[KO * 2], gy_re = acc[KO * 2 + 2];
  if (a.m0_lin) {
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) acc[v] = fma(t.y, a.m0_lin[v], acc[v]);
    if (GRAD) gy_re += a.m0_lin[0];
  }
  if (a.m0_const) {
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) acc[v] += a.m0_const[v];
  }
  if (a.out_re) {
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      double* dst = a.out_re + l * KO + k;
      *dst = a.accumulate ? *dst + acc[2 * k] : acc[2 * k];
    }
  }
  if (a.out_cplx) {
#pragma unroll
    for (int v = 0; v < KO * 2; ++v) {
      double* dst = a.out_cplx + l * KO * 2 + v;
      *dst = a.accumulate ? *dst + acc[v] : acc[v];
    }
  }
  if (GRAD && a.out_grad) {
    double* g = a.out_grad + 2 * l;
    g[0] = a.accumulate ? g[0] + gx_re : gx_re;
    g[1] = a.accumulate ? g[1] + gy_re : gy_re;
  }
}

void launch_chunk_sum(const double* partial, int chunks, size_t len, double* raw, cudaStream_t st) {
  if (len == 0) return;
  chunk_sum_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, st>>>(partial, chunks, len, raw);
  count_launches(1);
}

void launch_prep(const PrepArgs& a, cudaStream_t st) {
  if (a.count == 0) return;
  prep_kernel<<<(a.count + 127) / 128, 128, 0, st>>>(a);
  count_launches(1);
}

void launch_pw2t(const Pw2tArgs& a, cudaStream_t st) {
  if (a.nt == 0) return;
  const unsigned grid = static_cast<unsigned>((a.nt + kPw2tThreads - 1) / kPw2tThreads);
  const bool hasb = a.B != nullptr;
  count_launches(1);
  int dev = 0, sms = 148;
  cuda_check(cudaGetDevice(&dev), "device");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  if (grid < static_cast<unsigned>(sms) && a.modes.count >= 16) {  // fewer blocks than SMs: warps per target
    // a warp per target leaves ~7 warps per SM at c1's 1000 targets, each walking ~40 modes
    // serially; four warps per target (one target per block) when that still fills the GPU
    // with at most ~16 blocks per SM
    const bool wide = a.nt <= static_cast<size_t>(16) * sms && a.modes.count >= 4 * 32 * 4;
    auto go = [&](auto g) {
      constexpr int Gv = decltype(g)::value;
      const unsigned wgrid = static_cast<unsigned>((a.nt * 32 * Gv + kPw2tThreads - 1) / kPw2tThreads);
      if (a.ko == 1) {
        if (a.gradient)
          pw2t_warp_kernel<1, false, true, Gv><<<wgrid, kPw2tThreads, 0, st>>>(a);
        else if (hasb)
          pw2t_warp_kernel<1, true, false, Gv><<<wgrid, kPw2tThreads, 0, st>>>(a);
        else
          pw2t_warp_kernel<1, false, false, Gv><<<wgrid, kPw2tThreads, 0, st>>>(a);
      } else {
        if (hasb)
          pw2t_warp_kernel<2, true, false, Gv><<<wgrid, kPw2tThreads, 0, st>>>(a);
        else
          pw2t_warp_kernel<2, false, false, Gv><<<wgrid, kPw2tThreads, 0, st>>>(a);
      }
    };
    if (wide)
      go(std::integral_constant<int, 4>{});
    else
      go(std::integral_constant<int, 1>{});
    return;
  }
  if (a.ko == 1) {
    if (a.gradient)
      pw2t_kernel<1, false, true><<<grid, kPw2tThreads, 0, st>>>(a);
    else if (hasb)
      pw2t_kernel<1, true, false><<<grid, kPw2tThreads, 0, st>>>(a);
    else
      pw2t_kernel<1, false, false><<<grid, kPw2tThreads, 0, st>>>(a);
  } else {
    if (hasb)
      pw2t_kernel<2, true, false><<<grid, kPw2tThreads, 0, st>>>(a);
    else
      pw2t_kernel<2, false, false><<<grid, kPw2tThreads, 0, st>>>(a);
  }
}

void launch_reduce(const ReduceArgs& a, double* block_moments, double* block_checks, int blocks, cudaStream_t st) {
  reduce_kernel<<<blocks, kRedThreads, 0, st>>>(a, block_moments, block_checks);
  count_launches(1);
}

void launch_sum_blocks(const double* block_vals, int blocks, int n, double* out, cudaStream_t st) {
  sum_blocks_kernel<<<1, 32 * n, 0, st>>>(block_vals, blocks, n, out);
  count_launches(1);
}

}  // namespace pwb
