// Device NUFFT building blocks (nufft.cu) shared by the public transforms and the
// accelerated far-field routes of the engine.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "engine.hpp"
#include "periwave/periwave.hpp"
#include "pw_engine.cuh"

namespace pwb {

struct EsSpec {
  int w = 3;
  double beta = 6.9;
};
EsSpec es_spec(double eps);
size_t next_fast_even(size_t n);
size_t grid_size_for_modes(size_t nmodes, const EsSpec& s);
double phihat(const EsSpec& s, double xi);
std::vector<double> deconv_factors(const EsSpec& s, size_t nf, size_t nmodes);

// horizontal type-3 route (accel_h.cu)
struct HmixArgs {
  int nr = 0, lines = 0, stride = 0;  // F is [lines][stride], the part's modes start at f_off
  int f_off = 0;
  const double *decay_s = nullptr, *shift_s = nullptr, *decay_t = nullptr, *shift_t = nullptr;
  const double* diag = nullptr;
  const double* nodes = nullptr;
  const double* lam = nullptr;  // lambda_r of the part (target-side spread positions)
  double inv_h = 1.0, beta = 0.0;
  int nf = 0, w = 0;
};
struct HtgtArgs {
  size_t nt = 0;
  const double2* tgt = nullptr;
  double lo = 0.0, hi = 0.0;
  int lines = 0;
  double tk[kMaxLines] = {}, bw[kMaxLines] = {};
  double hx = 1.0;
  int nf = 0, w = 0, ngl = 0;
  const double* gl_amp = nullptr;
  const double* gl_z = nullptr;
};
void launch_hmix(const HmixArgs& a, const double* F, double* A, cudaStream_t st);
void launch_lam_spread(const HmixArgs& a, const double* A, double* g, cudaStream_t st);
void launch_htarget(const HtgtArgs& a, const double* g, double* out_re, double* out_cplx, cudaStream_t st);

int spread_lines_per_block(int nf, int lines);
void launch_spread(SpreadArgs a, double* grid_out, DevBuf& partial_ws, int sms, cudaStream_t st);
void launch_interp(const SpreadArgs& a, const double* grid, double* out_re, double* out_cplx, bool accumulate,
                   cudaStream_t st);
void launch_deconv(const double* grid, int lines, int nf, int nmodes, const double* fac, double* f, cudaStream_t st);
void launch_precorrect(const double* f, int lines, int nf, int nmodes, const double* fac, double* grid,
                       cudaStream_t st);
void launch_mix(const MixArgs& a, const double* F, double* G, cudaStream_t st);
void launch_exact_lines(const double* g, int lines, int nf, const double* s, int ns, double hx, const double* fac3,
                        double* f, cudaStream_t st);

}  // namespace pwb
