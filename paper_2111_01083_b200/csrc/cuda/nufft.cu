// NUFFT entry points (pwb_nufft_type1/2/3). Conventions of
// /root/reference/proj/include/periwave/nufft.hpp:10-18:
//   type1: f[k] = sum_j c[j] e^{+i k x[j]},  k = -(n/2) .. n-1-(n/2)
//   type2: c[j] = sum_k f[k] e^{-i k x[j]}
//   type3: f[k] = sum_j c[j] e^{+i s[k] x[j]}
// The Reference backend is the exact O(NM) sum (nufft.cpp:21-51), one thread
// per output with a fixed summation order.
#include <cuda_runtime.h>

#include "engine.hpp"
#include "periwave_b200.h"

namespace pwb {
namespace {

// out[i] = sum_j c[j] e^{i sign freq(i) pos(j)}; freq/pos: either integer modes or an array.
__global__ void exact_sum_kernel(size_t nout, size_t nin, const double* pos_in, const double* cin, long kmin_out,
                                 const double* freq_out, int sign, double* out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nout) return;
  const double fi = freq_out ? freq_out[i] : static_cast<double>(kmin_out + static_cast<long>(i));
  double re = 0.0, im = 0.0;
  for (size_t j = 0; j < nin; ++j) {
    double s, c;
    sincos(sign * fi * pos_in[j], &s, &c);
    const double a = cin[2 * j], b = cin[2 * j + 1];
    re += a * c - b * s;
    im += a * s + b * c;
  }
  out[2 * i] = re;
  out[2 * i + 1] = im;
}

// type 2: c[j] = sum_k f[k] e^{-i k x_j}; one thread per point.
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

struct Scoped {
  void* p = nullptr;
  ~Scoped() {
    if (p) cudaFree(p);
  }
};

const double* to_dev(Scoped& s, const double* h, size_t n, int memory) {
  if (memory == PWB_MEM_DEVICE || !h) return h;
  cuda_check(cudaMalloc(&s.p, (n + 1) * sizeof(double)), "cudaMalloc");
  if (n) cuda_check(cudaMemcpy(s.p, h, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
  return static_cast<const double*>(s.p);
}

}  // namespace

int nufft_entry(int type, int backend, double eps, size_t n, const double* x, const double* c, size_t nk,
                const double* s, double* f, int memory, void* stream) {
  (void)eps;
  if (backend == PWB_NUFFT_ACCELERATED)
    periwave::fail(periwave::ErrorCode::Unsupported, "accelerated NUFFT backend not built in this version");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw CudaFailure("no CUDA device available");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scoped sx, sc, ss, sf;
  const size_t nin = (type == 2) ? 2 * nk : 2 * n;
  const size_t nout = (type == 2) ? 2 * n : 2 * nk;
  const double* dx = to_dev(sx, x, n, memory);
  const double* dc = to_dev(sc, c, nin, memory);
  const double* ds = type == 3 ? to_dev(ss, s, nk, memory) : nullptr;
  double* df = f;
  if (memory != PWB_MEM_DEVICE) {
    cuda_check(cudaMalloc(&sf.p, (nout + 1) * sizeof(double)), "cudaMalloc");
    df = static_cast<double*>(sf.p);
  }
  if (type == 2) {
    if (n) exact_type2_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(n, dx, nk, dc, df);
  } else {
    const long kmin = -static_cast<long>(nk / 2);
    if (nk) exact_sum_kernel<<<static_cast<unsigned>((nk + 127) / 128), 128, 0, st>>>(nk, n, dx, dc, kmin, ds, 1, df);
  }
  cuda_check(cudaGetLastError(), "nufft launch");
  if (memory != PWB_MEM_DEVICE && nout)
    cuda_check(cudaMemcpyAsync(f, df, nout * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "nufft sync");
  return PWB_OK;
}

}  // namespace pwb
