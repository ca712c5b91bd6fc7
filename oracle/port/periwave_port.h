/* TEST INFRASTRUCTURE -- the CPU restatement used as a CHECKER and as the
 * "port" CPU baseline; never linked into or called by the product.
 *
 * Plain-C restatement of the reference's hot path (file:line per function in
 * periwave_port.c). Pinned against the compiled reference (oracle/_ref) in
 * tests/test_oracle_pins.py. Complex arrays are interleaved (re, im).
 */
#ifndef PERIWAVE_PORT_H
#define PERIWAVE_PORT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PORT_LAPLACE = 0, PORT_MODHELM = 1, PORT_STOKES = 2, PORT_MODSTOKES = 3, PORT_MULTIPOLE_LAPLACE = 4,
       PORT_MULTIPOLE_MODHELM = 5, PORT_STRESSLET = 6 };

/* modified Bessel K_l(x), own evaluation (series / trapezoidal integral) */
double port_bessel_kn(int l, double x);
/* xorshift64* uniform stream of the reference Rng (proj/include/periwave/util.hpp:83-98). */
void port_rng_uniform(unsigned long long seed, size_t n, double* out);

/* Near images: out += sum_img sum_j G((t_l - s_j) - shift_img) w_j, with the
 * reference's exact-zero rules (apply.cpp:481-546). Output per target:
 *   LAPLACE/MODHELM: 1 (+2 gradient if with_gradient, MODHELM only)
 *   STOKES/MODSTOKES: 2 (+1 pressure if with_pressure)
 *   MULTIPOLE_*: 2 (complex), STRESSLET: 2.
 * vec = forces or complex coefficients; nrm = normals (stresslet).
 * Returns 1 if a non-identity image coincided (CoincidentSourceTarget), else 0. */
int port_near(int kind, double beta, int order, size_t ns, const double* src, const double* q, const double* vec,
              const double* nrm, size_t nt, const double* tgt, int nimg, const double* shifts, int id_img,
              int with_pressure, int with_gradient, double* out, int nthreads);

/* One scalar part's direct apply into a complex accumulator (apply.cpp:45-78):
 * acc_l += sum_r T_l(r) diag_r sum_j S_j(r) w_j, plus m0 (vertical parts).
 * w: complex strengths. grad (nullable): complex d/dx, d/dy accumulators. */
void port_far_scalar(size_t nr, int axis, const double* phase, const double* dt, const double* ds, const double* st,
                     const double* ss, const double* diag, int has_m0, double m0_coef, size_t ns, const double* src,
                     const double* w, size_t nt, const double* tgt, double* acc, double* grad, int nthreads);

/* One block part (apply.cpp:80-118) into a Vec2c accumulator (4 doubles/target). */
void port_far_block(size_t nr, int axis, const double* phase, const double* dt, const double* ds, const double* st,
                    const double* ss, const double* diag_a, const double* diag_b, int three_term, int has_m0,
                    const double* m0_mat, size_t ns, const double* src, const double* f, size_t nt,
                    const double* tgt, double* acc, int nthreads);

/* Exact NUFFT sums (nufft.cpp:21-51). */
void port_nufft_type1(size_t n, const double* x, const double* c, size_t nmodes, double* f);
void port_nufft_type2(size_t n, const double* x, size_t nmodes, const double* f, double* c);
void port_nufft_type3(size_t n, const double* x, const double* c, size_t nk, const double* s, double* f);

#ifdef __cplusplus
}
#endif

#endif
