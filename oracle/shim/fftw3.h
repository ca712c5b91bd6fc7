/* TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
 *
 * FFTW3-shaped complex 1-D transform used by the reference's fast NUFFT
 * (/root/reference/proj/src/nufft_fast.cpp:7, :66-80). FFTW3 is absent from
 * the image and unpinned (/root/reference/proj/CMakeLists.txt:14-15). The
 * published contract reproduced here: unnormalised DFT,
 *   out[k] = sum_m in[m] exp(sign * 2 pi i k m / n),
 * with FFTW_FORWARD = -1 and FFTW_BACKWARD = +1. Implementation (own mixed
 * radix 2/3/5 recursion with a direct-DFT fallback for other factors) is in
 * oracle/shim/fftw_shim.cpp.
 */
#ifndef ORACLE_SHIM_FFTW3_H
#define ORACLE_SHIM_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct oracle_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
