// TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
//
// Stand-in for the three FFTW3 calls of /root/reference/proj/src/nufft_fast.cpp:66-80:
// an unnormalised complex DFT of any length, out[k] = sum_m in[m] e^{sign 2 pi i k m / n}.
// Decimation in time over the smallest prime factor (2, 3, 5 first; the
// reference only asks for 5-smooth lengths, nufft_fast.cpp:54-64), direct DFT for
// any remaining prime. Twiddles are formed from exact integer phases (k*r mod n)
// so the error stays O(log n) ulps.
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "fftw3.h"

namespace {

using cplx = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Plan {
  int n;
  int sign;
  cplx* in;
  cplx* out;
};

cplx twiddle(long num, long n, int sign) {
  long m = num % n;
  if (m < 0) m += n;
  return std::polar(1.0, sign * kTwoPi * static_cast<double>(m) / static_cast<double>(n));
}

void dft_rec(const cplx* x, long n, long stride, int sign, cplx* y) {
  if (n == 1) {
    y[0] = x[0];
    return;
  }
  long p = 0;
  for (long f : {2L, 3L, 5L})
    if (n % f == 0) {
      p = f;
      break;
    }
  if (p == 0) {
    for (long f = 7; f * f <= n; f += 2)
      if (n % f == 0) {
        p = f;
        break;
      }
  }
  if (p == 0) {  // prime length: direct sum
    for (long k = 0; k < n; ++k) {
      cplx acc{0.0, 0.0};
      for (long m = 0; m < n; ++m) acc += x[m * stride] * twiddle(k * m, n, sign);
      y[k] = acc;
    }
    return;
  }
  const long q = n / p;
  std::vector<cplx> sub(static_cast<size_t>(n));
  for (long r = 0; r < p; ++r) dft_rec(x + r * stride, q, stride * p, sign, sub.data() + r * q);
  for (long k = 0; k < q; ++k)
    for (long s = 0; s < p; ++s) {
      const long kk = k + s * q;
      cplx acc{0.0, 0.0};
      for (long r = 0; r < p; ++r) acc += sub[static_cast<size_t>(r * q + k)] * twiddle(r * kk, n, sign);
      y[kk] = acc;
    }
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned) {
  Plan* p = new Plan{n, sign >= 0 ? 1 : -1, reinterpret_cast<cplx*>(in), reinterpret_cast<cplx*>(out)};
  return reinterpret_cast<fftw_plan>(p);
}

void fftw_execute(const fftw_plan plan) {
  const Plan* p = reinterpret_cast<const Plan*>(plan);
  if (p->n <= 0) return;
  std::vector<cplx> src(p->in, p->in + p->n);
  dft_rec(src.data(), p->n, 1, p->sign, p->out);
}

void fftw_destroy_plan(fftw_plan plan) { delete reinterpret_cast<Plan*>(plan); }

}  // extern "C"
