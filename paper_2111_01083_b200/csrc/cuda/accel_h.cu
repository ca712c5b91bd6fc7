// Accelerated horizontal far field of singly periodic cells: the type-3 route of
// /root/reference/proj/src/apply.cpp:261-348 (fast_type3, nufft_fast.cpp:166-207).
//
// Per west/east part, with Legendre lines x_k on the cell's x interval:
//   source side  F_k[r] = sum_j gamma_k(x_j) q_j e^{-i lambda_r y_j}      (type 3, y -> -lambda)
//   mixing       a_k[r] = diag_r (sum_k' e^{ds_r (x_k' - ss_r)} F_k'[r]) e^{dt_r (x_k - st_r)}
//   target side  v_k(y) = sum_r a_k[r] e^{+i lambda_r y}                    (type 3, lambda -> y)
//                u_l   += sum_k gamma_k(x_l) v_k(y_l)
// Each type 3 spreads onto an open grid u_m = (m - nf/2) hx (ES kernel) and
// evaluates the small grid sum exactly; the deconvolution is (2/w)/phihat(s w hx/2).
// The source-side spreading reuses nufft.cu; the target side is one fused kernel
// (phasor recurrence over the nf2 grid points of every line, barycentric sum and
// the per-target deconvolution) so nothing of size lines x N is written.
#include <cuda_runtime.h>

#include "nufft.hpp"
#include "pw_engine.cuh"

namespace pwb {
namespace {

__global__ void hmix_kernel(const HmixArgs a, const double* F, double* A) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nr) return;
  const double ds = a.decay_s[r], ss = a.shift_s[r], dt = a.decay_t[r], st = a.shift_t[r];
  double sr = 0.0, si = 0.0;
  for (int k = 0; k < a.lines; ++k) {
    const double ex = exp(ds * (a.nodes[k] - ss));
    const size_t fi = (static_cast<size_t>(k) * a.stride + a.f_off + r) * 2;
    sr = fma(ex, F[fi], sr);
    si = fma(ex, F[fi + 1], si);
  }
  const double dr = a.diag[2 * r], di = a.diag[2 * r + 1];
  const double tr = dr * sr - di * si, ti = dr * si + di * sr;
  for (int k = 0; k < a.lines; ++k) {
    const double ex = exp(dt * (a.nodes[k] - st));
    A[(static_cast<size_t>(k) * a.nr + r) * 2] = tr * ex;
    A[(static_cast<size_t>(k) * a.nr + r) * 2 + 1] = ti * ex;
  }
}

// target-side spread of the nr frequencies lambda_r with line strengths a_k[r] onto
// the open grid of nf2 points: one thread per (line, grid point), fixed order.
__global__ void lam_spread_kernel(const HmixArgs a, const double* A, double* g) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (m >= a.nf || k >= a.lines) return;
  double gr = 0.0, gi = 0.0;
  const double sc = 2.0 / a.w;
  for (int r = 0; r < a.nr; ++r) {
    const double t = a.lam[r] * a.inv_h + 0.5 * a.nf;
    const long i0 = static_cast<long>(ceil(t - 0.5 * a.w));
    const long p = m - i0;
    if (p < 0 || p >= a.w) continue;
    const double z = (t - static_cast<double>(m)) * sc;
    const double q = 1.0 - z * z;
    if (q <= 0.0) continue;
    const double phi = exp(a.beta * (sqrt(q) - 1.0));
    gr = fma(A[(static_cast<size_t>(k) * a.nr + r) * 2], phi, gr);
    gi = fma(A[(static_cast<size_t>(k) * a.nr + r) * 2 + 1], phi, gi);
  }
  g[(static_cast<size_t>(k) * a.nf + m) * 2] = gr;
  g[(static_cast<size_t>(k) * a.nf + m) * 2 + 1] = gi;
}

__device__ __forceinline__ double bary_w(const HtgtArgs& a, double t, int k, int hit, double inv) {
  if (hit >= 0) return k == hit ? 1.0 : 0.0;
  return a.bw[k] / (t - a.tk[k]) * inv;
}

// u_l += [sum_k gamma_k(x_l) sum_m g_k[m] e^{+i (m - nf/2) y_l hx}] (2/w)/phihat(y_l w hx/2)
__global__ void htarget_kernel(const HtgtArgs a, const double* g, double* out_re, double* out_cplx) {
  const size_t l = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= a.nt) return;
  const double2 p = a.tgt[l];
  // barycentric row in x (quadrature.cpp:283-304)
  const double t = (2.0 * p.x - a.lo - a.hi) / (a.hi - a.lo);
  int hit = -1;
  double sum = 0.0;
  for (int k = 0; k < a.lines; ++k) {
    const double d = t - a.tk[k];
    if (d == 0.0) {
      hit = k;
      break;
    }
    sum += a.bw[k] / d;
  }
  const double inv = hit >= 0 ? 0.0 : 1.0 / sum;
  const double th = p.y * a.hx;
  double s1, c1, s0, c0;
  sincos(th, &s1, &c1);
  sincos(-0.5 * a.nf * th, &s0, &c0);
  double vr = 0.0, vi = 0.0;
  for (int k = 0; k < a.lines; ++k) {
    const double wk = bary_w(a, t, k, hit, inv);
    if (wk == 0.0) continue;
    const double* line = g + static_cast<size_t>(k) * a.nf * 2;
    double er = c0, ei = s0, ir = 0.0, ii = 0.0;
    for (int m = 0; m < a.nf; ++m) {
      const double gr = line[2 * m], gi = line[2 * m + 1];
      ir = fma(gr, er, fma(-gi, ei, ir));
      ii = fma(gr, ei, fma(gi, er, ii));
      const double nr = er * c1 - ei * s1;
      ei = fma(er, s1, ei * c1);
      er = nr;
    }
    vr = fma(wk, ir, vr);
    vi = fma(wk, ii, vi);
  }
  // phihat(y w hx / 2) from the (3w+20)-point rule (nufft_fast.cpp:45-52)
  const double xi = p.y * 0.5 * a.w * a.hx;
  double ps = 0.0;
  for (int i = 0; i < a.ngl; ++i) ps = fma(a.gl_amp[i], cos(xi * a.gl_z[i]), ps);
  const double f = (2.0 / a.w) / ps;
  if (out_re) out_re[l] += vr * f;
  if (out_cplx) {
    out_cplx[2 * l] += vr * f;
    out_cplx[2 * l + 1] += vi * f;
  }
}

}  // namespace

void launch_hmix(const HmixArgs& a, const double* F, double* A, cudaStream_t st) {
  if (a.nr == 0) return;
  hmix_kernel<<<(a.nr + 127) / 128, 128, 0, st>>>(a, F, A);
  count_launches(1);
}

void launch_lam_spread(const HmixArgs& a, const double* A, double* g, cudaStream_t st) {
  lam_spread_kernel<<<dim3((a.nf + 127) / 128, a.lines), 128, 0, st>>>(a, A, g);
  count_launches(1);
}

void launch_htarget(const HtgtArgs& a, const double* g, double* out_re, double* out_cplx, cudaStream_t st) {
  if (a.nt == 0) return;
  htarget_kernel<<<static_cast<unsigned>((a.nt + 127) / 128), 128, 0, st>>>(a, g, out_re, out_cplx);
  count_launches(1);
}

}  // namespace pwb
