/* TEST INFRASTRUCTURE -- CPU restatement of the reference hot path (checker /
 * "port" CPU baseline only; the product never loads this file).
 *
 * Follows /root/reference/proj/src/apply.cpp and kernels.cpp function by
 * function (file:line cited below). Deliberately simple scalar loops in
 * reference order; pthreads split the target loop like parallel_for
 * (util.hpp:61-79), so results are independent of the thread count.
 */
#include "periwave_port.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define PORT_PI 3.14159265358979323846264338327950288
#define EULER_G 0.57721566490153286060651209008240243

/* ------------------------------------------------------------------ Bessel K_l
 * kernels.cpp:78-96 (GSL scaled K times e^{-x}, underflow -> 0). Own evaluation:
 * ascending series for x <= 2 (A&S 9.6.13/9.6.11), trapezoidal rule on
 * K_n(x) = int_0^inf e^{-x cosh t} cosh(n t) dt for x > 2. */
static void series01(double x, double* k0, double* k1) {
  const double t = 0.25 * x * x, lh = log(0.5 * x);
  double i0 = 0, s0 = 0, i1 = 0, s1 = 0, a = 1, b = 1, h = 0;
  for (int k = 0; k < 40; ++k) {
    i0 += a;
    s0 += h * a;
    i1 += b;
    const double h1 = h + 1.0 / (k + 1.0);
    s1 += (h + h1 - 2.0 * EULER_G) * b;
    a *= t / ((k + 1.0) * (k + 1.0));
    b *= t / ((k + 1.0) * (k + 2.0));
    h = h1;
    if (a < 1e-19 * i0 && b < 1e-19 * i1) break;
  }
  *k0 = -(lh + EULER_G) * i0 + s0;
  *k1 = 1.0 / x + lh * 0.5 * x * i1 - 0.25 * x * s1;
}

static double trap_k(int n, double x) {
  /* step ~ 1/sqrt(x) (Gaussian width), cosh t - 1 = 2 sinh^2(t/2) without cancellation */
  const double hstep = fmin(0.125, 0.5 / sqrt(x));
  double acc = 0.5;
  for (int k = 1; k < 100000; ++k) {
    const double t = k * hstep, sh = sinh(0.5 * t), a = 2.0 * x * sh * sh;
    acc += n == 0 ? exp(-a) : exp(-a) * cosh(n * t);
    if (a - n * t > 45.0) break;
  }
  return hstep * acc * exp(-x);
}

double port_bessel_kn(int l, double x) {
  if (!(x > 0.0)) return NAN;
  if (x > 700.0) return 0.0;
  double k0, k1;
  if (x <= 2.0) {
    series01(x, &k0, &k1);
  } else {
    k0 = trap_k(0, x);
    k1 = trap_k(1, x);
  }
  if (l == 0) return k0;
  double km = k0, kc = k1;
  for (int i = 1; i < l; ++i) {
    const double kn = km + (2.0 * i / x) * kc;
    km = kc;
    kc = kn;
  }
  return kc;
}

/* kernels.cpp:40-68: g1 = 1 - z K1, g2 = -1 + z K1 + z^2 K0, series for z < 0.5 */
static void g12(double z, double* g1, double* g2) {
  if (z >= 0.5) {
    const double zk1 = z * port_bessel_kn(1, z);
    *g1 = 1.0 - zk1;
    *g2 = -*g1 + z * z * port_bessel_kn(0, z);
    return;
  }
  const double q = 0.25 * z * z, lg = log(0.5 * z);
  double i0 = 0, i1 = 0, s0 = 0, s1 = 0, term = 1, psi = -EULER_G;
  for (int k = 0; k < 18; ++k) {
    i0 += term;
    i1 += term / (k + 1.0);
    s0 += term * psi;
    const double pn = psi + 1.0 / (k + 1.0);
    s1 += term * (psi + pn) / (k + 1.0);
    psi = pn;
    term *= q / ((k + 1.0) * (k + 1.0));
    if (term < 1e-20) break;
  }
  i1 *= 0.5 * z;
  const double k0 = -lg * i0 + s0;
  *g1 = -z * lg * i1 + q * s1;
  *g2 = -*g1 + z * z * k0;
}

/* ------------------------------------------------------------------ near images */
typedef struct {
  int kind, order, nimg, id_img, with_pressure, with_gradient, nout;
  double beta;
  size_t ns, nt, lo, hi;
  const double *src, *q, *vec, *nrm, *tgt, *shifts;
  double* out;
  int coincident;
} near_job;

static int near_nout(int kind, int with_pressure, int with_gradient) {
  switch (kind) {
    case PORT_LAPLACE: return 1;
    case PORT_MODHELM: return with_gradient ? 3 : 1;
    case PORT_STOKES:
    case PORT_MODSTOKES: return with_pressure ? 3 : 2;
    default: return 2;
  }
}

/* apply.cpp:493-543 with greens_scalar / greens_block / multipole_kernel / stresslet_dlp */
static void* near_worker(void* arg) {
  near_job* J = (near_job*)arg;
  const double c_st = -1.0 / (4.0 * PORT_PI);
  for (size_t l = J->lo; l < J->hi; ++l) {
    const double tx = J->tgt[2 * l], ty = J->tgt[2 * l + 1];
    double* o = J->out + l * (size_t)J->nout;
    for (int im = 0; im < J->nimg; ++im) {
      const double shx = J->shifts[2 * im], shy = J->shifts[2 * im + 1];
      double u[3] = {0, 0, 0};
      for (size_t j = 0; j < J->ns; ++j) {
        const double rx = (tx - J->src[2 * j]) - shx, ry = (ty - J->src[2 * j + 1]) - shy;
        if (rx == 0.0 && ry == 0.0) {
          if (im != J->id_img) J->coincident = 1;
          continue;
        }
        const double r2 = rx * rx + ry * ry, rr = hypot(rx, ry);
        switch (J->kind) {
          case PORT_LAPLACE: u[0] += -log(rr) / (2.0 * PORT_PI) * J->q[j]; break;
          case PORT_MODHELM: {
            const double x = J->beta * rr;
            u[0] += port_bessel_kn(0, x) / (2.0 * PORT_PI) * J->q[j];
            if (J->with_gradient) {
              const double g = -J->beta / (2.0 * PORT_PI) * port_bessel_kn(1, x) / rr * J->q[j];
              u[1] += g * rx;
              u[2] += g * ry;
            }
            break;
          }
          case PORT_STOKES: {
            const double lg = 0.5 * log(r2), fx = J->vec[2 * j], fy = J->vec[2 * j + 1];
            const double a11 = c_st * (lg - rx * rx / r2), a12 = c_st * (-rx * ry / r2), a22 = c_st * (lg - ry * ry / r2);
            u[0] += a11 * fx + a12 * fy;
            u[1] += a12 * fx + a22 * fy;
            if (J->with_pressure) u[2] += rx / (2.0 * PORT_PI * r2) * fx + ry / (2.0 * PORT_PI * r2) * fy;
            break;
          }
          case PORT_MODSTOKES: {
            double g1, g2;
            g12(J->beta * sqrt(r2), &g1, &g2);
            const double c = 1.0 / (2.0 * PORT_PI * J->beta * J->beta * r2);
            const double xh2 = rx * rx / r2, yh2 = ry * ry / r2, xy = rx * ry / r2;
            const double a11 = c * (g2 * yh2 + g1 * xh2), a12 = -c * xy * (g2 - g1), a22 = c * (g2 * xh2 + g1 * yh2);
            const double fx = J->vec[2 * j], fy = J->vec[2 * j + 1];
            u[0] += a11 * fx + a12 * fy;
            u[1] += a12 * fx + a22 * fy;
            if (J->with_pressure) u[2] += rx / (2.0 * PORT_PI * r2) * fx + ry / (2.0 * PORT_PI * r2) * fy;
            break;
          }
          case PORT_MULTIPOLE_LAPLACE:
          case PORT_MULTIPOLE_MODHELM: {
            double pr = 1, pi = 0, vr, vi;
            if (J->kind == PORT_MULTIPOLE_LAPLACE) {
              for (int k = 0; k < J->order; ++k) {
                const double t = pr * rx - pi * ry;
                pi = pr * ry + pi * rx;
                pr = t;
              }
              const double dd = pr * pr + pi * pi;
              vr = pr / dd;
              vi = -pi / dd;
            } else {
              const double kl = port_bessel_kn(J->order, J->beta * rr);
              for (int k = 0; k < J->order; ++k) {
                const double t = pr * (rx / rr) - pi * (ry / rr);
                pi = pr * (ry / rr) + pi * (rx / rr);
                pr = t;
              }
              vr = kl * pr;
              vi = kl * pi;
            }
            const double cr = J->vec[2 * j], ci = J->vec[2 * j + 1];
            u[0] += vr * cr - vi * ci;
            u[1] += vr * ci + vi * cr;
            break;
          }
          case PORT_STRESSLET: {
            const double nx = J->nrm[2 * j], ny = J->nrm[2 * j + 1];
            const double c = -(rx * nx + ry * ny) / (PORT_PI * r2 * r2);
            const double fx = J->vec[2 * j], fy = J->vec[2 * j + 1];
            u[0] += c * rx * rx * fx + c * rx * ry * fy;
            u[1] += c * rx * ry * fx + c * ry * ry * fy;
            break;
          }
        }
      }
      for (int c = 0; c < J->nout; ++c) o[c] += u[c];
    }
  }
  return NULL;
}

int port_near(int kind, double beta, int order, size_t ns, const double* src, const double* q, const double* vec,
              const double* nrm, size_t nt, const double* tgt, int nimg, const double* shifts, int id_img,
              int with_pressure, int with_gradient, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  near_job jobs[256];
  pthread_t th[256];
  const size_t chunk = (nt + nthreads - 1) / (size_t)nthreads;
  int started = 0;
  for (int w = 0; w < nthreads; ++w) {
    near_job* J = &jobs[w];
    memset(J, 0, sizeof *J);
    J->kind = kind;
    J->order = order;
    J->nimg = nimg;
    J->id_img = id_img;
    J->with_pressure = with_pressure;
    J->with_gradient = with_gradient;
    J->nout = near_nout(kind, with_pressure, with_gradient);
    J->beta = beta;
    J->ns = ns;
    J->nt = nt;
    J->lo = w * chunk < nt ? w * chunk : nt;
    J->hi = J->lo + chunk < nt ? J->lo + chunk : nt;
    J->src = src;
    J->q = q;
    J->vec = vec;
    J->nrm = nrm;
    J->tgt = tgt;
    J->shifts = shifts;
    J->out = out;
    if (nthreads == 1)
      near_worker(J);
    else if (pthread_create(&th[w], NULL, near_worker, J) == 0)
      started = w + 1;
    else
      near_worker(J);
  }
  for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
  int coincident = 0;
  for (int w = 0; w < nthreads; ++w) coincident |= jobs[w].coincident;
  return coincident;
}

/* ------------------------------------------------------------------ far field (direct)
 * Mode factors apply.cpp:32-38; vertical parts w = y, p = x; horizontal w = x, p = y. */
static void src_factor(double ph, double ds, double ss, double w, double p, double* re, double* im) {
  const double m = exp(ds * (w - ss));
  *re = m * cos(-ph * p);
  *im = m * sin(-ph * p);
}

typedef struct {
  size_t nr, ns, lo, hi, kstr;
  int axis, three_term, grad;
  const double *phase, *dt, *ds, *st, *ss, *src, *w, *tgt;
  const double* coef;  /* per-mode complex target coefficients */
  const double* coefb; /* block: second (w-weighted) coefficient set */
  double *acc, *gacc;
  int block;
} far_job;

static void* far_target_worker(void* arg) {
  far_job* J = (far_job*)arg;
  for (size_t l = J->lo; l < J->hi; ++l) {
    const double x = J->tgt[2 * l], y = J->tgt[2 * l + 1];
    const double w = J->axis ? x : y, p = J->axis ? y : x;
    double u[4] = {0, 0, 0, 0}, gx[2] = {0, 0}, gy[2] = {0, 0};
    for (size_t r = 0; r < J->nr; ++r) {
      const double m = exp(J->dt[r] * (w - J->st[r]));
      const double tr = m * cos(J->phase[r] * p), ti = m * sin(J->phase[r] * p);
      if (!J->block) {
        const double cr = J->coef[2 * r], ci = J->coef[2 * r + 1];
        const double pr = tr * cr - ti * ci, pi = tr * ci + ti * cr;
        u[0] += pr;
        u[1] += pi;
        if (J->grad) {
          const double ir = -J->phase[r] * pi, ii = J->phase[r] * pr, dr = J->dt[r] * pr, di = J->dt[r] * pi;
          if (J->axis) {
            gx[0] += dr; gx[1] += di; gy[0] += ir; gy[1] += ii;
          } else {
            gx[0] += ir; gx[1] += ii; gy[0] += dr; gy[1] += di;
          }
        }
      } else {
        /* u0 = D_a s1 (+ D_b s2 - w D_b s1), apply.cpp:101-105 */
        for (int c = 0; c < 2; ++c) {
          double cr = J->coef[4 * r + 2 * c], ci = J->coef[4 * r + 2 * c + 1];
          if (J->three_term) {
            cr -= w * J->coefb[4 * r + 2 * c];
            ci -= w * J->coefb[4 * r + 2 * c + 1];
          }
          u[2 * c] += tr * cr - ti * ci;
          u[2 * c + 1] += tr * ci + ti * cr;
        }
      }
    }
    const int nc = J->block ? 4 : 2;
    for (int c = 0; c < nc; ++c) J->acc[l * nc + c] += u[c];
    if (J->grad && J->gacc) {
      J->gacc[4 * l] += gx[0];
      J->gacc[4 * l + 1] += gx[1];
      J->gacc[4 * l + 2] += gy[0];
      J->gacc[4 * l + 3] += gy[1];
    }
  }
  return NULL;
}

static void run_targets(far_job* base, size_t nt, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  far_job jobs[256];
  pthread_t th[256];
  const size_t chunk = (nt + nthreads - 1) / (size_t)nthreads;
  int started = 0;
  for (int w = 0; w < nthreads; ++w) {
    jobs[w] = *base;
    jobs[w].lo = w * chunk < nt ? w * chunk : nt;
    jobs[w].hi = jobs[w].lo + chunk < nt ? jobs[w].lo + chunk : nt;
    if (nthreads == 1)
      far_target_worker(&jobs[w]);
    else if (pthread_create(&th[w], NULL, far_target_worker, &jobs[w]) == 0)
      started = w + 1;
    else
      far_target_worker(&jobs[w]);
  }
  for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
}

/* apply.cpp:45-78 */
void port_far_scalar(size_t nr, int axis, const double* phase, const double* dt, const double* ds, const double* st,
                     const double* ss, const double* diag, int has_m0, double m0_coef, size_t ns, const double* src,
                     const double* w, size_t nt, const double* tgt, double* acc, double* grad, int nthreads) {
  double* coef = (double*)calloc(2 * nr + 2, sizeof(double));
  for (size_t r = 0; r < nr; ++r) {
    double sr = 0, si = 0;
    for (size_t j = 0; j < ns; ++j) {
      double fr, fi;
      const double wc = axis ? src[2 * j] : src[2 * j + 1], pc = axis ? src[2 * j + 1] : src[2 * j];
      src_factor(phase[r], ds[r], ss[r], wc, pc, &fr, &fi);
      sr += fr * w[2 * j] - fi * w[2 * j + 1];
      si += fr * w[2 * j + 1] + fi * w[2 * j];
    }
    coef[2 * r] = diag[2 * r] * sr - diag[2 * r + 1] * si;
    coef[2 * r + 1] = diag[2 * r] * si + diag[2 * r + 1] * sr;
  }
  far_job J;
  memset(&J, 0, sizeof J);
  J.nr = nr;
  J.axis = axis;
  J.grad = grad != NULL;
  J.phase = phase;
  J.dt = dt;
  J.st = st;
  J.tgt = tgt;
  J.coef = coef;
  J.acc = acc;
  J.gacc = grad;
  run_targets(&J, nt, nthreads);
  if (has_m0) { /* apply.cpp:68-78, vertical parts: w = y */
    double mr = 0, mi = 0;
    for (size_t j = 0; j < ns; ++j) {
      const double wc = axis ? src[2 * j] : src[2 * j + 1];
      mr += wc * w[2 * j];
      mi += wc * w[2 * j + 1];
    }
    mr *= m0_coef;
    mi *= m0_coef;
    for (size_t l = 0; l < nt; ++l) {
      const double wc = axis ? tgt[2 * l] : tgt[2 * l + 1];
      acc[2 * l] += wc * mr;
      acc[2 * l + 1] += wc * mi;
      if (grad && !axis) {
        grad[4 * l + 2] += mr;
        grad[4 * l + 3] += mi;
      }
    }
  }
  free(coef);
}

/* apply.cpp:80-118 */
void port_far_block(size_t nr, int axis, const double* phase, const double* dt, const double* ds, const double* st,
                    const double* ss, const double* diag_a, const double* diag_b, int three_term, int has_m0,
                    const double* m0_mat, size_t ns, const double* src, const double* f, size_t nt,
                    const double* tgt, double* acc, int nthreads) {
  double* ca = (double*)calloc(4 * nr + 4, sizeof(double));
  double* cb = (double*)calloc(4 * nr + 4, sizeof(double));
  for (size_t r = 0; r < nr; ++r) {
    double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    for (size_t j = 0; j < ns; ++j) {
      double fr, fi;
      const double wc = axis ? src[2 * j] : src[2 * j + 1], pc = axis ? src[2 * j + 1] : src[2 * j];
      src_factor(phase[r], ds[r], ss[r], wc, pc, &fr, &fi);
      const double v[4] = {fr * f[2 * j], fi * f[2 * j], fr * f[2 * j + 1], fi * f[2 * j + 1]};
      for (int k = 0; k < 4; ++k) {
        s1[k] += v[k];
        if (three_term) s2[k] += wc * v[k];
      }
    }
    const double* A = diag_a + 8 * r;
    const double* B = diag_b ? diag_b + 8 * r : NULL;
    for (int row = 0; row < 2; ++row) {
      double ar = 0, ai = 0, br = 0, bi = 0;
      for (int col = 0; col < 2; ++col) {
        const double mr = A[4 * row + 2 * col], mi = A[4 * row + 2 * col + 1];
        ar += mr * s1[2 * col] - mi * s1[2 * col + 1];
        ai += mr * s1[2 * col + 1] + mi * s1[2 * col];
        if (three_term && B) {
          const double nr_ = B[4 * row + 2 * col], ni = B[4 * row + 2 * col + 1];
          ar += nr_ * s2[2 * col] - ni * s2[2 * col + 1];
          ai += nr_ * s2[2 * col + 1] + ni * s2[2 * col];
          br += nr_ * s1[2 * col] - ni * s1[2 * col + 1];
          bi += nr_ * s1[2 * col + 1] + ni * s1[2 * col];
        }
      }
      ca[4 * r + 2 * row] = ar;
      ca[4 * r + 2 * row + 1] = ai;
      cb[4 * r + 2 * row] = br;
      cb[4 * r + 2 * row + 1] = bi;
    }
  }
  far_job J;
  memset(&J, 0, sizeof J);
  J.nr = nr;
  J.axis = axis;
  J.block = 1;
  J.three_term = three_term;
  J.phase = phase;
  J.dt = dt;
  J.st = st;
  J.tgt = tgt;
  J.coef = ca;
  J.coefb = cb;
  J.acc = acc;
  run_targets(&J, nt, nthreads);
  if (has_m0) {
    double mx = 0, my = 0;
    for (size_t j = 0; j < ns; ++j) {
      const double wc = axis ? src[2 * j] : src[2 * j + 1];
      mx += f[2 * j] * wc;
      my += f[2 * j + 1] * wc;
    }
    const double bx = m0_mat[0] * mx + m0_mat[1] * my, by = m0_mat[2] * mx + m0_mat[3] * my;
    for (size_t l = 0; l < nt; ++l) {
      const double wc = axis ? tgt[2 * l] : tgt[2 * l + 1];
      acc[4 * l] += wc * bx;
      acc[4 * l + 2] += wc * by;
    }
  }
  free(ca);
  free(cb);
}

/* ------------------------------------------------------------------ exact NUFFT sums (nufft.cpp:21-51) */
void port_nufft_type1(size_t n, const double* x, const double* c, size_t nmodes, double* f) {
  const long kmin = -(long)(nmodes / 2);
  memset(f, 0, 2 * nmodes * sizeof(double));
  for (size_t j = 0; j < n; ++j)
    for (size_t k = 0; k < nmodes; ++k) {
      const double a = (double)(kmin + (long)k) * x[j];
      const double cr = cos(a), ci = sin(a);
      f[2 * k] += c[2 * j] * cr - c[2 * j + 1] * ci;
      f[2 * k + 1] += c[2 * j] * ci + c[2 * j + 1] * cr;
    }
}

void port_nufft_type2(size_t n, const double* x, size_t nmodes, const double* f, double* c) {
  const long kmin = -(long)(nmodes / 2);
  for (size_t j = 0; j < n; ++j) {
    double re = 0, im = 0;
    for (size_t k = 0; k < nmodes; ++k) {
      const double a = -(double)(kmin + (long)k) * x[j];
      const double cr = cos(a), ci = sin(a);
      re += f[2 * k] * cr - f[2 * k + 1] * ci;
      im += f[2 * k] * ci + f[2 * k + 1] * cr;
    }
    c[2 * j] = re;
    c[2 * j + 1] = im;
  }
}

void port_nufft_type3(size_t n, const double* x, const double* c, size_t nk, const double* s, double* f) {
  for (size_t k = 0; k < nk; ++k) {
    double re = 0, im = 0;
    for (size_t j = 0; j < n; ++j) {
      const double a = s[k] * x[j];
      const double cr = cos(a), ci = sin(a);
      re += c[2 * j] * cr - c[2 * j + 1] * ci;
      im += c[2 * j] * ci + c[2 * j + 1] * cr;
    }
    f[2 * k] = re;
    f[2 * k + 1] = im;
  }
}

/* xorshift64* step mapped to [0, 1), restating proj/include/periwave/util.hpp:83-98
   (seed 0 is replaced by the golden-ratio constant, as upstream). */
void port_rng_uniform(unsigned long long seed, size_t n, double* out) {
  unsigned long long s = seed ? seed : 0x9e3779b97f4a7c15ull;
  for (size_t i = 0; i < n; ++i) {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    out[i] = (double)((s * 0x2545f4914f6cdd1dull) >> 11) * 0x1.0p-53;
  }
}
