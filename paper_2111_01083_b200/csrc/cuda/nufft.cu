// NUFFT on the device: exponential-of-semicircle spreading / interpolation,
// cuFFT for the uniform transforms, deconvolution, and the barycentric line
// machinery of the accelerated far field.
//
// Conventions (/root/reference/proj/include/periwave/nufft.hpp:10-18):
//   type1: f[k] = sum_j c[j] e^{+i k x[j]},  k = -(n/2) .. n-1-(n/2)
//   type2: c[j] = sum_k f[k] e^{-i k x[j]}
//   type3: f[k] = sum_j c[j] e^{+i s[k] x[j]}
// Accelerated backend restates /root/reference/proj/src/nufft_fast.cpp:
//   ES kernel phi(z) = exp(beta (sqrt(1 - z^2) - 1)), w = clamp(ceil(log10 1/eps) + 1, 3, 16),
//   beta = 2.3 w (:26-40); grid nf = 5-smooth even >= max(2 n, 2w + 4) (:54-64, :127-130);
//   t = remainder(x, 2 pi)/h, taps i0 = ceil(t - w/2) + p, z = (t - tap)(2/w) (:82-114);
//   deconvolution by (2/w)/phihat(k w h / 2), phihat by a (3w+20)-point Gauss-Legendre rule
//   (:45-52, :124-164); type 3 = spread on the open grid u_m = (m - nf/2) hx, hx = pi/(2 smax),
//   then a type-2 evaluation at -s hx and deconvolution (:166-207).
// Spreading accumulates per block in shared memory (fp64 atomics), blocks write
// per-chunk partial grids that are summed in a fixed order. The Reference backend
// is the exact O(NM) sum (nufft.cpp:21-51), one thread per output.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "nufft.hpp"
#include "periwave_b200.h"

namespace pwb {

// ---------------------------------------------------------------- host side parameters
EsSpec es_spec(double eps) {  // nufft_fast.cpp:36-40
  eps = std::min(std::max(eps, 1e-14), 1e-2);
  EsSpec s;
  s.w = std::min(std::max(static_cast<int>(std::ceil(std::log10(1.0 / eps))) + 1, 3), 16);
  s.beta = 2.30 * s.w;
  return s;
}

size_t next_fast_even(size_t n) {  // nufft_fast.cpp:54-64
  if (n < 2) n = 2;
  if (n % 2) ++n;
  for (;; n += 2) {
    size_t m = n;
    while (m % 2 == 0) m /= 2;
    while (m % 3 == 0) m /= 3;
    while (m % 5 == 0) m /= 5;
    if (m == 1) return n;
  }
}

size_t grid_size_for_modes(size_t nmodes, const EsSpec& s) {  // nufft_fast.cpp:127-130
  return next_fast_even(std::max<size_t>(static_cast<size_t>(std::ceil(2.0 * static_cast<double>(nmodes))),
                                         static_cast<size_t>(2 * s.w + 4)));
}

// integral of phi(z) e^{-i xi z} over [-1, 1] (real, even): (3w+20)-point GL (nufft_fast.cpp:45-52)
double phihat(const EsSpec& s, double xi) {
  static std::mutex mu;
  static std::map<int, periwave::GaussRule> cache;
  const periwave::GaussRule* g;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(s.w);
    if (it == cache.end()) it = cache.emplace(s.w, periwave::gauss_legendre(3 * s.w + 20)).first;
    g = &it->second;
  }
  double acc = 0.0;
  for (size_t i = 0; i < g->nodes.size(); ++i) {
    const double z = g->nodes[i];
    const double t = 1.0 - z * z;
    const double phi = t <= 0.0 ? 0.0 : std::exp(s.beta * (std::sqrt(t) - 1.0));
    acc += g->weights[i] * phi * std::cos(xi * z);
  }
  return acc;
}

// (2/w)/phihat(k w h / 2) for the modes kmin .. kmin+n-1 on a grid of nf points
std::vector<double> deconv_factors(const EsSpec& s, size_t nf, size_t nmodes) {
  std::vector<double> out(nmodes);
  const double h = 2.0 * periwave::kPi / static_cast<double>(nf);
  const long kmin = -static_cast<long>(nmodes / 2);
  for (size_t i = 0; i < nmodes; ++i) {
    const long kk = kmin + static_cast<long>(i);
    out[i] = (2.0 / s.w) / phihat(s, static_cast<double>(kk) * 0.5 * s.w * h);
  }
  return out;
}

namespace {

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ long es_taps(double t, int w, double beta, double* phi) {
  const long i0 = static_cast<long>(ceil(t - 0.5 * w));
  const double sc = 2.0 / w;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    if (p < w) {
      const double z = (t - static_cast<double>(i0 + p)) * sc;
      const double q = 1.0 - z * z;
      phi[p] = q <= 0.0 ? 0.0 : exp(beta * (sqrt(q) - 1.0));
    } else {
      phi[p] = 0.0;
    }
  }
  return i0;
}

__device__ __forceinline__ int wrap_index(long m, long nf) {
  long r = m % nf;
  if (r < 0) r += nf;
  return static_cast<int>(r);
}

// Barycentric interpolation row at coordinate v (quadrature.cpp:283-304): exact node
// hit -> one-hot, else w_k/(t - t_k) normalised. Returns the row entry for `k`
// given the precomputed denominator (or the one-hot index).
struct BaryRow {
  int hit;       // node index on an exact hit, else -1
  double tnorm;  // t of the point
  double inv;    // 1 / sum_k w_k/(t - t_k)
};

__device__ __forceinline__ BaryRow bary_row(const BaryGrid& g, double v) {
  BaryRow b;
  b.tnorm = (2.0 * v - g.lo - g.hi) / (g.hi - g.lo);
  b.hit = -1;
  double sum = 0.0;
  for (int k = 0; k < g.m; ++k) {
    const double d = b.tnorm - g.tk[k];
    if (d == 0.0) {
      b.hit = k;
      break;
    }
    sum += g.bw[k] / d;
  }
  b.inv = b.hit >= 0 ? 0.0 : 1.0 / sum;
  return b;
}

__device__ __forceinline__ double bary_entry(const BaryGrid& g, const BaryRow& b, int k) {
  if (b.hit >= 0) return k == b.hit ? 1.0 : 0.0;
  return g.bw[k] / (b.tnorm - g.tk[k]) * b.inv;
}

// position of a point on the spreading grid
__device__ __forceinline__ double grid_t(const SpreadArgs& a, double p) {
  if (a.open) return p * a.inv_h + 0.5 * static_cast<double>(a.nf);
  return remainder(p, 2.0 * 3.14159265358979323846) / a.h;
}

__device__ __forceinline__ double point_pos(const SpreadArgs& a, size_t j, double2* bary_coord) {
  switch (a.pos) {
    case PosKind::WrappedX: {  // -wrap_to_rectangle(p).x * 2 pi / d (apply.cpp:219, cell.cpp:72-75)
      const double2 p = a.pts[j];
      *bary_coord = p;
      const double k = floor(p.x / a.d + 0.5);
      return -(p.x - k * a.d) * a.kx;
    }
    case PosKind::PointY: {
      const double2 p = a.pts[j];
      *bary_coord = p;
      return p.y;
    }
    default:
      *bary_coord = make_double2(0.0, 0.0);
      return a.xs[j];
  }
}

__device__ __forceinline__ double bary_coord_of(const SpreadArgs& a, double2 p) {
  return a.bary_axis == 0 ? p.y : p.x;
}

__device__ __forceinline__ void strength_of(const SpreadArgs& a, size_t j, double* re, double* im) {
  if (a.cplx) {
    *re = a.c[2 * j];
    *im = a.c[2 * j + 1];
  } else {
    *re = a.c[j];
    *im = 0.0;
  }
}

// ---------------------------------------------------------------- spreading
// grid z = blockIdx.y: line group; blockIdx.x: point chunk. Shared grid [lpg][nf][2].
__global__ void spread_kernel(const __grid_constant__ SpreadArgs a, double* partial) {
  extern __shared__ double sg[];
  const int g = blockIdx.y;
  const int k0 = g * a.lpg;
  const int kn = min(a.lines - k0, a.lpg);
  const int nf = a.nf;
  for (int i = threadIdx.x; i < kn * nf * 2; i += blockDim.x) sg[i] = 0.0;
  __syncthreads();
  const size_t j0 = static_cast<size_t>(blockIdx.x) * a.per_chunk;
  const size_t j1 = min(a.n, j0 + a.per_chunk);
  for (size_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    double2 bc;
    const double p = point_pos(a, j, &bc);
    const double t = grid_t(a, p);
    double phi[16];
    const long i0 = es_taps(t, a.w, a.beta, phi);
    double cr, ci;
    strength_of(a, j, &cr, &ci);
    BaryRow br;
    const bool bary = a.bary.m > 0;
    if (bary) br = bary_row(a.bary, bary_coord_of(a, bc));
    for (int kk = 0; kk < kn; ++kk) {
      const double row = bary ? bary_entry(a.bary, br, k0 + kk) : 1.0;
      if (row == 0.0) continue;
      const double vr = row * cr, vi = row * ci;
      double* line = sg + static_cast<size_t>(kk) * nf * 2;
      for (int q = 0; q < a.w; ++q) {
        const int m = a.open ? static_cast<int>(i0 + q) : wrap_index(i0 + q, nf);
        atomicAdd(line + 2 * m, vr * phi[q]);
        atomicAdd(line + 2 * m + 1, vi * phi[q]);
      }
    }
  }
  __syncthreads();
  double* dst = partial + (static_cast<size_t>(blockIdx.x) * a.lines + k0) * nf * 2;
  for (int i = threadIdx.x; i < kn * nf * 2; i += blockDim.x) dst[i] = sg[i];
}

__global__ void chunk_reduce_kernel(const double* partial, int chunks, size_t len, double* out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= len) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += partial[static_cast<size_t>(c) * len + i];
  out[i] = s;
}

// ---------------------------------------------------------------- interpolation
// out_j (+)= sum_k row_k(point) sum_p grid_k[tap_p] phi_p   (complex)
__global__ void interp_kernel(const __grid_constant__ SpreadArgs a, const double* grid, double* out_re,
                              double* out_cplx, int accumulate) {
  const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  double2 bc;
  const double p = point_pos(a, j, &bc);
  const double t = grid_t(a, p);
  double phi[16];
  const long i0 = es_taps(t, a.w, a.beta, phi);
  int idx[16];
#pragma unroll
  for (int q = 0; q < 16; ++q)
    idx[q] = q < a.w ? (a.open ? static_cast<int>(i0 + q) : wrap_index(i0 + q, a.nf)) : 0;
  BaryRow br;
  const bool bary = a.bary.m > 0;
  if (bary) br = bary_row(a.bary, bary_coord_of(a, bc));
  double ur = 0.0, ui = 0.0;
  for (int k = 0; k < a.lines; ++k) {
    const double row = bary ? bary_entry(a.bary, br, k) : 1.0;
    if (row == 0.0) continue;
    const double* line = grid + static_cast<size_t>(k) * a.nf * 2;
    double vr = 0.0, vi = 0.0;
    for (int q = 0; q < a.w; ++q) {
      const double2 gv = *reinterpret_cast<const double2*>(line + 2 * idx[q]);
      vr = fma(gv.x, phi[q], vr);
      vi = fma(gv.y, phi[q], vi);
    }
    ur = fma(row, vr, ur);
    ui = fma(row, vi, ui);
  }
  if (out_re) out_re[j] = accumulate ? out_re[j] + ur : ur;
  if (out_cplx) {
    out_cplx[2 * j] = accumulate ? out_cplx[2 * j] + ur : ur;
    out_cplx[2 * j + 1] = accumulate ? out_cplx[2 * j + 1] + ui : ui;
  }
}

// ---------------------------------------------------------------- uniform-mode steps
// type 1 deconvolution: f[k][i] = grid[k][wrap(kmin+i)] * fac[i]
__global__ void deconv_kernel(const double* grid, int lines, int nf, int nmodes, const double* fac, double* f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= nmodes || k >= lines) return;
  const long kk = -static_cast<long>(nmodes / 2) + i;
  const int m = wrap_index(kk, nf);
  const double2 v = *reinterpret_cast<const double2*>(grid + (static_cast<size_t>(k) * nf + m) * 2);
  f[(static_cast<size_t>(k) * nmodes + i) * 2] = v.x * fac[i];
  f[(static_cast<size_t>(k) * nmodes + i) * 2 + 1] = v.y * fac[i];
}

// type 2 precorrection: grid[k][wrap(kmin+i)] = f[k][i] * fac[i] (grid zeroed before)
__global__ void precorrect_kernel(const double* f, int lines, int nf, int nmodes, const double* fac, double* grid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= nmodes || k >= lines) return;
  const long kk = -static_cast<long>(nmodes / 2) + i;
  const int m = wrap_index(kk, nf);
  grid[(static_cast<size_t>(k) * nf + m) * 2] = f[(static_cast<size_t>(k) * nmodes + i) * 2] * fac[i];
  grid[(static_cast<size_t>(k) * nf + m) * 2 + 1] = f[(static_cast<size_t>(k) * nmodes + i) * 2 + 1] * fac[i];
}

// accelerated vertical mode mixing (apply.cpp:230-244): per mode index m, every mode r
// with that index in part order: s = diag_r sum_k e^{ds (y_k - ss)} F_k[m];
// G_k[m] += s e^{dt (y_k - st)}
__global__ void mix_kernel(const __grid_constant__ MixArgs a, const double* F, double* G) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.nmodes) return;
  double gr[64], gi[64];
  for (int k = 0; k < a.lines; ++k) gr[k] = gi[k] = 0.0;
  for (int e = a.bucket_start[m]; e < a.bucket_start[m + 1]; ++e) {
    const int r = a.bucket[e];
    const double ds = a.decay_s[r], ss = a.shift_s[r], dt = a.decay_t[r], st = a.shift_t[r];
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < a.lines; ++k) {
      const double ex = exp(ds * (a.nodes[k] - ss));
      sr = fma(ex, F[(static_cast<size_t>(k) * a.nmodes + m) * 2], sr);
      si = fma(ex, F[(static_cast<size_t>(k) * a.nmodes + m) * 2 + 1], si);
    }
    const double dr = a.diag[2 * r], di = a.diag[2 * r + 1];
    const double tr = dr * sr - di * si, ti = dr * si + di * sr;
    for (int k = 0; k < a.lines; ++k) {
      const double ex = exp(dt * (a.nodes[k] - st));
      gr[k] = fma(tr, ex, gr[k]);
      gi[k] = fma(ti, ex, gi[k]);
    }
  }
  for (int k = 0; k < a.lines; ++k) {
    G[(static_cast<size_t>(k) * a.nmodes + m) * 2] = gr[k];
    G[(static_cast<size_t>(k) * a.nmodes + m) * 2 + 1] = gi[k];
  }
}

// type-3 inner step (nufft_fast.cpp:521-531): f[k][i] = (sum_m g_k[m] e^{-i (m - nf/2) th_i})
// * fac3[i] where th_i = -s_i hx; evaluated by ES interpolation on the type-2 grid of the
// open-grid spread -- here exactly, one thread per (line, frequency): nf*w work is small.
__global__ void exact_lines_kernel(const double* g, int lines, int nf, const double* s, int ns, double hx,
                                   const double* fac3, double* f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= ns || k >= lines) return;
  double re = 0.0, im = 0.0;
  const double* line = g + static_cast<size_t>(k) * nf * 2;
  for (int m = 0; m < nf; ++m) {
    double sn, cs;
    sincos(s[i] * (m - 0.5 * nf) * hx, &sn, &cs);
    const double a = line[2 * m], b = line[2 * m + 1];
    re += a * cs - b * sn;
    im += a * sn + b * cs;
  }
  f[(static_cast<size_t>(k) * ns + i) * 2] = re * fac3[i];
  f[(static_cast<size_t>(k) * ns + i) * 2 + 1] = im * fac3[i];
}

// ---------------------------------------------------------------- exact sums (Reference backend)
__global__ void exact_sum_kernel(size_t nout, size_t nin, const double* pos_in, const double* cin, long kmin_out,
                                 const double* freq_out, double* out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nout) return;
  const double fi = freq_out ? freq_out[i] : static_cast<double>(kmin_out + static_cast<long>(i));
  double re = 0.0, im = 0.0;
  for (size_t j = 0; j < nin; ++j) {
    double s, c;
    sincos(fi * pos_in[j], &s, &c);
    const double a = cin[2 * j], b = cin[2 * j + 1];
    re += a * c - b * s;
    im += a * s + b * c;
  }
  out[2 * i] = re;
  out[2 * i + 1] = im;
}

__global__ void exact_type2_kernel(size_t n, const double* x, size_t nm, const double* f, double* c) {
  const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const long kmin = -static_cast<long>(nm / 2);
  double re = 0.0, im = 0.0;
  for (size_t k = 0; k < nm; ++k) {
    double s, cs;
    sincos(-static_cast<double>(kmin + static_cast<long>(k)) * x[j], &s, &cs);
    const double a = f[2 * k], b = f[2 * k + 1];
    re += a * cs - b * s;
    im += a * s + b * cs;
  }
  c[2 * j] = re;
  c[2 * j + 1] = im;
}

void fft_check(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) throw CudaFailure(std::string(what) + ": cuFFT error " + std::to_string(static_cast<int>(r)));
}

}  // namespace

// ---------------------------------------------------------------- launchers
int spread_lines_per_block(int nf, int lines) {
  const size_t per_line = static_cast<size_t>(nf) * 2 * sizeof(double);
  const size_t budget = 200 * 1024;
  int lpg = static_cast<int>(std::max<size_t>(1, budget / per_line));
  return std::min(lpg, lines);
}

void launch_spread(SpreadArgs a, double* grid_out, DevBuf& partial_ws, int sms, cudaStream_t st) {
  const size_t len = static_cast<size_t>(a.lines) * a.nf * 2;
  if (a.n == 0) {
    cuda_check(cudaMemsetAsync(grid_out, 0, len * sizeof(double), st), "memset grid");
    return;
  }
  a.lpg = spread_lines_per_block(a.nf, a.lines);
  const int groups = (a.lines + a.lpg - 1) / a.lpg;
  if (static_cast<size_t>(a.nf) * 2 * sizeof(double) > 200 * 1024)
    throw InternalFailure("spreading grid too large for shared memory");
  int chunks = std::max(1, (2 * sms + groups - 1) / groups);
  chunks = static_cast<int>(std::min<size_t>(chunks, std::max<size_t>(1, a.n / 256)));
  a.per_chunk = (a.n + chunks - 1) / chunks;
  double* partial = partial_ws.as<double>(static_cast<size_t>(chunks) * len);
  const size_t smem = static_cast<size_t>(a.lpg) * a.nf * 2 * sizeof(double);
  cuda_check(cudaFuncSetAttribute(spread_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "smem attribute");
  spread_kernel<<<dim3(chunks, groups), 512, smem, st>>>(a, partial);
  chunk_reduce_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, st>>>(partial, chunks, len, grid_out);
  count_launches(2);
}

void launch_interp(const SpreadArgs& a, const double* grid, double* out_re, double* out_cplx, bool accumulate,
                   cudaStream_t st) {
  if (a.n == 0) return;
  interp_kernel<<<static_cast<unsigned>((a.n + 127) / 128), 128, 0, st>>>(a, grid, out_re, out_cplx,
                                                                          accumulate ? 1 : 0);
  count_launches(1);
}

void launch_deconv(const double* grid, int lines, int nf, int nmodes, const double* fac, double* f, cudaStream_t st) {
  deconv_kernel<<<dim3((nmodes + 127) / 128, lines), 128, 0, st>>>(grid, lines, nf, nmodes, fac, f);
  count_launches(1);
}

void launch_precorrect(const double* f, int lines, int nf, int nmodes, const double* fac, double* grid,
                       cudaStream_t st) {
  cuda_check(cudaMemsetAsync(grid, 0, static_cast<size_t>(lines) * nf * 2 * sizeof(double), st), "memset grid");
  precorrect_kernel<<<dim3((nmodes + 127) / 128, lines), 128, 0, st>>>(f, lines, nf, nmodes, fac, grid);
  count_launches(1);
}

void launch_mix(const MixArgs& a, const double* F, double* G, cudaStream_t st) {
  if (a.lines > 64) throw InternalFailure("mode mixing supports at most 64 lines");
  mix_kernel<<<(a.nmodes + 127) / 128, 128, 0, st>>>(a, F, G);
  count_launches(1);
}

void launch_exact_lines(const double* g, int lines, int nf, const double* s, int ns, double hx, const double* fac3,
                        double* f, cudaStream_t st) {
  if (ns == 0) return;
  exact_lines_kernel<<<dim3((ns + 127) / 128, lines), 128, 0, st>>>(g, lines, nf, s, ns, hx, fac3, f);
  count_launches(1);
}

FftPlans::~FftPlans() {
  for (auto& kv : plans_) cufftDestroy(static_cast<cufftHandle>(kv.second));
}

void FftPlans::exec(double* data, int nf, int lines, int sign, cudaStream_t st) {
  auto key = std::make_pair(nf, lines);
  auto it = plans_.find(key);
  if (it == plans_.end()) {
    cufftHandle plan;
    int n[1] = {nf};
    fft_check(cufftPlanMany(&plan, 1, n, nullptr, 1, nf, nullptr, 1, nf, CUFFT_Z2Z, lines), "cufftPlanMany");
    it = plans_.emplace(key, static_cast<int>(plan)).first;
  }
  const cufftHandle plan = static_cast<cufftHandle>(it->second);
  fft_check(cufftSetStream(plan, st), "cufftSetStream");
  auto* z = reinterpret_cast<cufftDoubleComplex*>(data);
  fft_check(cufftExecZ2Z(plan, z, z, sign > 0 ? CUFFT_INVERSE : CUFFT_FORWARD), "cufftExecZ2Z");
  count_launches(1);
}

// ---------------------------------------------------------------- the public transforms
namespace {

struct Scoped {
  void* p = nullptr;
  ~Scoped() {
    if (p) cudaFree(p);
  }
};

const double* to_dev(Scoped& s, const double* h, size_t n, int memory, cudaStream_t st) {
  if (memory == PWB_MEM_DEVICE || !h) return h;
  cuda_check(cudaMalloc(&s.p, (n + 1) * sizeof(double)), "cudaMalloc");
  if (n) cuda_check(cudaMemcpyAsync(s.p, h, n * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
  return static_cast<const double*>(s.p);
}

double* upload_vec(Scoped& s, const std::vector<double>& v, cudaStream_t st) {
  cuda_check(cudaMalloc(&s.p, (v.size() + 1) * sizeof(double)), "cudaMalloc");
  if (!v.empty())
    cuda_check(cudaMemcpyAsync(s.p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
  return static_cast<double*>(s.p);
}

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

// type 1 (accelerated) on device arrays: x[n], c[n] complex, f[nmodes] complex
void fast_type1_dev(double eps, size_t n, const double* x, const double* c, size_t nmodes, double* f,
                    cudaStream_t st) {
  cuda_check(cudaMemsetAsync(f, 0, 2 * nmodes * sizeof(double), st), "memset");
  if (n == 0 || nmodes == 0) return;
  const EsSpec s = es_spec(eps);
  const size_t nf = grid_size_for_modes(nmodes, s);
  Scoped g, fac;
  cuda_check(cudaMalloc(&g.p, 2 * nf * sizeof(double)), "cudaMalloc");
  double* fac_d = upload_vec(fac, deconv_factors(s, nf, nmodes), st);
  SpreadArgs a;
  a.n = n;
  a.pos = PosKind::Array;
  a.xs = x;
  a.c = c;
  a.cplx = 1;
  a.nf = static_cast<int>(nf);
  a.h = 2.0 * periwave::kPi / static_cast<double>(nf);
  a.w = s.w;
  a.beta = s.beta;
  a.lines = 1;
  DevBuf ws;
  FftPlans fft;  // destroyed after the final synchronize below
  launch_spread(a, static_cast<double*>(g.p), ws, device_sms(), st);
  fft.exec(static_cast<double*>(g.p), static_cast<int>(nf), 1, +1, st);
  launch_deconv(static_cast<double*>(g.p), 1, static_cast<int>(nf), static_cast<int>(nmodes), fac_d, f, st);
  cuda_check(cudaStreamSynchronize(st), "sync");
}

// type 2 (accelerated): f[nmodes] complex -> c[n] complex at x[n]
void fast_type2_dev(double eps, size_t n, const double* x, size_t nmodes, const double* f, double* c,
                    cudaStream_t st) {
  cuda_check(cudaMemsetAsync(c, 0, 2 * n * sizeof(double), st), "memset");
  if (n == 0 || nmodes == 0) return;
  const EsSpec s = es_spec(eps);
  const size_t nf = grid_size_for_modes(nmodes, s);
  Scoped g, fac;
  cuda_check(cudaMalloc(&g.p, 2 * nf * sizeof(double)), "cudaMalloc");
  double* fac_d = upload_vec(fac, deconv_factors(s, nf, nmodes), st);
  FftPlans fft;  // destroyed after the final synchronize below
  launch_precorrect(f, 1, static_cast<int>(nf), static_cast<int>(nmodes), fac_d, static_cast<double*>(g.p), st);
  fft.exec(static_cast<double*>(g.p), static_cast<int>(nf), 1, -1, st);
  SpreadArgs a;
  a.n = n;
  a.pos = PosKind::Array;
  a.xs = x;
  a.nf = static_cast<int>(nf);
  a.h = 2.0 * periwave::kPi / static_cast<double>(nf);
  a.w = s.w;
  a.beta = s.beta;
  a.lines = 1;
  launch_interp(a, static_cast<double*>(g.p), nullptr, c, false, st);
  cuda_check(cudaStreamSynchronize(st), "sync");
}

// type 3 (accelerated): f[k] = sum_j c_j e^{i s_k x_j} (nufft_fast.cpp:166-207)
void fast_type3_dev(double eps, size_t n, const double* x_dev, const double* c, size_t nk, const double* s_dev,
                    double* f, cudaStream_t st, double xmax, double smax) {
  cuda_check(cudaMemsetAsync(f, 0, 2 * nk * sizeof(double), st), "memset");
  if (nk == 0 || n == 0) return;
  const EsSpec sp = es_spec(eps);
  const double hx = periwave::kPi / (2.0 * smax);
  const size_t nf = next_fast_even(2 * static_cast<size_t>(std::ceil(xmax / hx)) + 2 * sp.w + 4);
  periwave::require(nf <= (size_t{1} << 24), periwave::ErrorCode::Unsupported, "type-3 transform extent too large");
  Scoped g, fac;
  cuda_check(cudaMalloc(&g.p, 2 * nf * sizeof(double)), "cudaMalloc");
  SpreadArgs a;
  a.n = n;
  a.pos = PosKind::Array;
  a.xs = x_dev;
  a.c = c;
  a.cplx = 1;
  a.open = 1;
  a.inv_h = 1.0 / hx;
  a.nf = static_cast<int>(nf);
  a.w = sp.w;
  a.beta = sp.beta;
  a.lines = 1;
  DevBuf ws;
  launch_spread(a, static_cast<double*>(g.p), ws, device_sms(), st);
  // inner type 2 at -s hx (nufft_fast.cpp:521-526) done exactly on the open grid, then
  // deconvolution by (2/w)/phihat(s w hx / 2) (:527-531)
  std::vector<double> s_host(nk);
  cuda_check(cudaMemcpyAsync(s_host.data(), s_dev, nk * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  std::vector<double> fac3(nk);
  for (size_t i = 0; i < nk; ++i) fac3[i] = (2.0 / sp.w) / phihat(sp, s_host[i] * 0.5 * sp.w * hx);
  double* fac_d = upload_vec(fac, fac3, st);
  launch_exact_lines(static_cast<double*>(g.p), 1, static_cast<int>(nf), s_dev, static_cast<int>(nk), hx, fac_d, f,
                     st);
  cuda_check(cudaStreamSynchronize(st), "sync");
}

int nufft_entry(int type, int backend, double eps, size_t n, const double* x, const double* c, size_t nk,
                const double* s, double* f, int memory, void* stream) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw CudaFailure("no CUDA device available");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scoped sx, sc, ss, sf;
  const size_t nin = (type == 2) ? 2 * nk : 2 * n;
  const size_t nout = (type == 2) ? 2 * n : 2 * nk;
  const double* dx = to_dev(sx, x, n, memory, st);
  const double* dc = to_dev(sc, c, nin, memory, st);
  const double* ds = type == 3 ? to_dev(ss, s, nk, memory, st) : nullptr;
  double* df = f;
  if (memory != PWB_MEM_DEVICE) {
    cuda_check(cudaMalloc(&sf.p, (nout + 1) * sizeof(double)), "cudaMalloc");
    df = static_cast<double*>(sf.p);
  }
  if (backend == PWB_NUFFT_ACCELERATED) {
    if (type == 1) {
      fast_type1_dev(eps, n, dx, dc, nk, df, st);
    } else if (type == 2) {
      fast_type2_dev(eps, n, dx, nk, dc, df, st);
    } else {
      // extents from the host copies when available, else read back
      std::vector<double> hx(n), hs(nk);
      cuda_check(cudaMemcpyAsync(hx.data(), dx, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      cuda_check(cudaMemcpyAsync(hs.data(), ds, nk * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      cuda_check(cudaStreamSynchronize(st), "sync");
      double xmax = 0.0, smax = 0.0;
      for (double v : hx) xmax = std::max(xmax, std::abs(v));
      for (double v : hs) smax = std::max(smax, std::abs(v));
      if (xmax == 0.0 || smax == 0.0) {  // nufft_fast.cpp:498-503: every output is sum c
        std::vector<double> hc(2 * n);
        cuda_check(cudaMemcpyAsync(hc.data(), dc, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        double tr = 0.0, ti = 0.0;
        for (size_t j = 0; j < n; ++j) {
          tr += hc[2 * j];
          ti += hc[2 * j + 1];
        }
        std::vector<double> hf(2 * nk);
        for (size_t k = 0; k < nk; ++k) {
          hf[2 * k] = tr;
          hf[2 * k + 1] = ti;
        }
        cuda_check(cudaMemcpyAsync(df, hf.data(), 2 * nk * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
      } else if (n > 0 && nk > 0) {
        fast_type3_dev(eps, n, dx, dc, nk, ds, df, st, xmax, smax);
      } else {
        cuda_check(cudaMemsetAsync(df, 0, nout * sizeof(double), st), "memset");
      }
    }
  } else if (type == 2) {
    if (n) {
      exact_type2_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(n, dx, nk, dc, df);
      count_launches(1);
    }
  } else {
    const long kmin = -static_cast<long>(nk / 2);
    if (nk) {
      exact_sum_kernel<<<static_cast<unsigned>((nk + 127) / 128), 128, 0, st>>>(nk, n, dx, dc, kmin, ds, df);
      count_launches(1);
    }
  }
  cuda_check(cudaGetLastError(), "nufft launch");
  if (memory != PWB_MEM_DEVICE && nout)
    cuda_check(cudaMemcpyAsync(f, df, nout * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "nufft sync");
  return PWB_OK;
}

}  // namespace pwb
