// TEST INFRASTRUCTURE -- the CHECKER, never the product.
//
// extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/) so the
// Python test-suite and bench.py's CPU-baseline leg can call it through ctypes.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) load the resulting oracle/_ref/libperiwave_ref.so.
//
// Return convention: 0 on success, 1 + periwave::ErrorCode ordinal on a
// periwave::Error (/root/reference/proj/include/periwave/errors.hpp:8-28), -1 on
// any other exception; ref_last_error() holds the message.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "periwave/periwave.hpp"

using namespace periwave;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

UnitCell cell_of(double d, double xi, double eta, int periodicity) {
  return make_unit_cell(d, xi, eta, periodicity == 1 ? Periodicity::Singly : Periodicity::Doubly);
}

std::vector<Vec2> vec2s(const double* p, size_t n) {
  std::vector<Vec2> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = {p[2 * i], p[2 * i + 1]};
  return v;
}

ParticleSystem system_of(size_t ns, const double* src, const double* charges, const double* forces,
                         const double* normals, const double* coeffs, size_t nt, const double* tgt) {
  ParticleSystem s;
  if (src) s.sources = vec2s(src, ns);
  if (charges) s.charges.assign(charges, charges + ns);
  if (forces) s.forces = vec2s(forces, ns);
  if (normals) s.normals = vec2s(normals, ns);
  if (coeffs) {
    s.coefficients.resize(ns);
    for (size_t i = 0; i < ns; ++i) s.coefficients[i] = {coeffs[2 * i], coeffs[2 * i + 1]};
  }
  if (tgt) s.targets = vec2s(tgt, nt);
  return s;
}

ApplyOptions options_of(int path, int threads, int with_pressure, double nufft_eps) {
  ApplyOptions o;
  o.path = path == 1 ? ApplyPath::Direct : path == 2 ? ApplyPath::Accelerated : ApplyPath::Auto;
  o.threads = threads;
  o.with_pressure = with_pressure != 0;
  o.nufft_eps = nufft_eps;
  return o;
}

void export_field(const FieldResult& f, double* scalar, double* velocity, double* pressure,
                  double* cplx_out, int* accelerated) {
  if (scalar)
    for (size_t i = 0; i < f.scalar.size(); ++i) scalar[i] = f.scalar[i];
  if (velocity)
    for (size_t i = 0; i < f.velocity.size(); ++i) {
      velocity[2 * i] = f.velocity[i].x;
      velocity[2 * i + 1] = f.velocity[i].y;
    }
  if (pressure)
    for (size_t i = 0; i < f.pressure.size(); ++i) pressure[i] = f.pressure[i];
  if (cplx_out)
    for (size_t i = 0; i < f.complex_scalar.size(); ++i) {
      cplx_out[2 * i] = f.complex_scalar[i].real();
      cplx_out[2 * i + 1] = f.complex_scalar[i].imag();
    }
  if (accelerated) *accelerated = f.accelerated ? 1 : 0;
}

FieldResult import_field(const Periodizer& pz, size_t nt, const double* scalar, const double* velocity,
                         const double* pressure, const double* cplx_in) {
  FieldResult f;
  if (pz.multipole_order >= 1) {
    f.complex_scalar.resize(nt);
    for (size_t i = 0; i < nt; ++i) f.complex_scalar[i] = {cplx_in[2 * i], cplx_in[2 * i + 1]};
  } else if (pz.pde == Pde::Stokes || pz.pde == Pde::ModStokes) {
    f.velocity = vec2s(velocity, nt);
    if (pressure) f.pressure.assign(pressure, pressure + nt);
  } else {
    f.scalar.assign(scalar, scalar + nt);
  }
  return f;
}

void put_cplx(const std::vector<cplx>& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

void put_mat2c(const std::vector<Mat2c>& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    const cplx e[4] = {v[i].a11, v[i].a12, v[i].a21, v[i].a22};
    for (int k = 0; k < 4; ++k) {
      out[8 * i + 2 * k] = e[k].real();
      out[8 * i + 2 * k + 1] = e[k].imag();
    }
  }
}

const ModeSet* modes_of(const Periodizer& pz, int kind, int idx) {
  switch (kind) {
    case 0: return &pz.scalar_parts.at(idx).modes;
    case 1: return &pz.block_parts.at(idx).modes;
    case 2: return &pz.pressure_parts.at(idx).modes;
    default: return &pz.stresslet_parts.at(idx).modes;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// The reference's own periwave::Rng stream (util.hpp:83-98): the bench's reference arm
// draws its inputs from it, so that arm never loads the product library.
void ref_rng_uniform(unsigned long long seed, size_t n, double* out) {
  periwave::Rng r(seed);
  for (size_t i = 0; i < n; ++i) out[i] = r.uniform();
}

int ref_unit_cell_m0(double d, double xi, double eta, int periodicity, int* m0) {
  return guarded([&] { *m0 = cell_of(d, xi, eta, periodicity).m0; });
}

void* ref_make_periodizer(int pde, double beta, double d, double xi, double eta, int periodicity, double eps,
                          int* err) {
  Periodizer* out = nullptr;
  *err = guarded([&] { out = new Periodizer(make_periodizer(static_cast<Pde>(pde), beta, cell_of(d, xi, eta, periodicity), eps)); });
  return out;
}

void* ref_make_multipole_periodizer(int pde, double beta, int l, double d, double xi, double eta,
                                    int periodicity, double eps, int* err) {
  Periodizer* out = nullptr;
  *err = guarded([&] {
    out = new Periodizer(make_multipole_periodizer(static_cast<Pde>(pde), beta, l, cell_of(d, xi, eta, periodicity), eps));
  });
  return out;
}

void* ref_make_stokes_dlp_periodizer(double d, double xi, double eta, int periodicity, double eps, int* err) {
  Periodizer* out = nullptr;
  *err = guarded([&] { out = new Periodizer(make_stokes_dlp_periodizer(cell_of(d, xi, eta, periodicity), eps)); });
  return out;
}

void ref_free_periodizer(void* pz) { delete static_cast<Periodizer*>(pz); }

size_t ref_rank(void* pz) { return static_cast<Periodizer*>(pz)->rank(); }

int ref_requires_neutrality(void* pz) { return static_cast<Periodizer*>(pz)->requires_neutrality ? 1 : 0; }

// kind: 0 scalar, 1 block, 2 pressure, 3 stresslet
int ref_num_parts(void* p, int kind) {
  const Periodizer& pz = *static_cast<Periodizer*>(p);
  switch (kind) {
    case 0: return static_cast<int>(pz.scalar_parts.size());
    case 1: return static_cast<int>(pz.block_parts.size());
    case 2: return static_cast<int>(pz.pressure_parts.size());
    default: return static_cast<int>(pz.stresslet_parts.size());
  }
}

// info[0] axis, info[1] dir, info[2] take_real/three_term, info[3] has_m0, info[4] size;
// m0[0..3] m0_coef or m0_mat entries (pressure: coef, row.x, row.y)
int ref_part_info(void* p, int kind, int idx, long* info, double* m0) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    const ModeSet& ms = *modes_of(pz, kind, idx);
    info[0] = static_cast<long>(ms.axis);
    info[4] = static_cast<long>(ms.size());
    for (int k = 0; k < 4; ++k) m0[k] = 0.0;
    if (kind == 0) {
      const ScalarPart& s = pz.scalar_parts.at(idx);
      info[1] = static_cast<long>(s.dir);
      info[2] = s.take_real;
      info[3] = s.has_m0;
      m0[0] = s.m0_coef;
    } else if (kind == 1) {
      const BlockPart& b = pz.block_parts.at(idx);
      info[1] = static_cast<long>(b.dir);
      info[2] = b.three_term;
      info[3] = b.has_m0;
      m0[0] = b.m0_mat.a11;
      m0[1] = b.m0_mat.a12;
      m0[2] = b.m0_mat.a21;
      m0[3] = b.m0_mat.a22;
    } else if (kind == 2) {
      const PressurePart& q = pz.pressure_parts.at(idx);
      info[1] = static_cast<long>(q.dir);
      info[2] = 0;
      info[3] = q.has_m0;
      m0[0] = q.m0_coef;
      m0[1] = q.m0_row.x;
      m0[2] = q.m0_row.y;
    } else {
      const StressletPart& q = pz.stresslet_parts.at(idx);
      info[1] = static_cast<long>(q.dir);
      info[2] = 0;
      info[3] = q.has_m0;
      m0[0] = q.m0_coef;
    }
  });
}

int ref_part_modes(void* p, int kind, int idx, double* phase, double* decay_t, double* decay_s, double* shift_t,
                   double* shift_s) {
  return guarded([&] {
    const ModeSet& ms = *modes_of(*static_cast<Periodizer*>(p), kind, idx);
    for (size_t r = 0; r < ms.size(); ++r) {
      phase[r] = ms.phase[r];
      decay_t[r] = ms.decay_t[r];
      decay_s[r] = ms.decay_s[r];
      shift_t[r] = ms.shift_t[r];
      shift_s[r] = ms.shift_s[r];
    }
  });
}

// which: scalar {0 diag}; block {0 diag_a, 1 diag_b}; pressure {0 diag, 1 row};
// stresslet {0 a1, 1 a2, 2 smat, 3 sa, 4 sb, 5 off}. Complex values interleaved
// (re, im); Mat2c as 4 complex row-major; Vec2c as 2 complex.
int ref_part_table(void* p, int kind, int idx, int which, double* out) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    if (kind == 0) {
      put_cplx(pz.scalar_parts.at(idx).diag, out);
    } else if (kind == 1) {
      const BlockPart& b = pz.block_parts.at(idx);
      put_mat2c(which == 0 ? b.diag_a : b.diag_b, out);
    } else if (kind == 2) {
      const PressurePart& q = pz.pressure_parts.at(idx);
      if (which == 0) {
        put_cplx(q.diag, out);
      } else {
        for (size_t r = 0; r < q.row.size(); ++r) {
          out[4 * r] = q.row[r].x.real();
          out[4 * r + 1] = q.row[r].x.imag();
          out[4 * r + 2] = q.row[r].y.real();
          out[4 * r + 3] = q.row[r].y.imag();
        }
      }
    } else {
      const StressletPart& q = pz.stresslet_parts.at(idx);
      switch (which) {
        case 0: put_mat2c(q.a1, out); break;
        case 1: put_mat2c(q.a2, out); break;
        case 2: put_mat2c(q.smat, out); break;
        case 3: put_cplx(q.sa, out); break;
        case 4: put_cplx(q.sb, out); break;
        default: put_cplx(q.off, out); break;
      }
    }
  });
}

// mode: 0 total_field, 1 apply_far, 2 near images only (sum over near_translations)
int ref_apply(void* p, int mode, size_t ns, const double* src, const double* charges, const double* forces,
              const double* normals, const double* coeffs, size_t nt, const double* tgt, int path, int threads,
              int with_pressure, double nufft_eps, double* scalar, double* velocity, double* pressure,
              double* cplx_out, int* accelerated) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    ParticleSystem sys = system_of(ns, src, charges, forces, normals, coeffs, nt, tgt);
    ApplyOptions opt = options_of(path, threads, with_pressure, nufft_eps);
    FieldResult f;
    if (mode == 0) {
      f = total_field(pz, sys, opt);
    } else if (mode == 1) {
      f = apply_far(pz, sys, opt);
    } else {
      FreeSpaceEvaluator ev;
      for (const LatticeTranslation& tr : near_translations(pz.cell))
        ev.accumulate(pz, sys, tr.shift, tr.m == 0 && tr.n == 0, opt, f);
    }
    export_field(f, scalar, velocity, pressure, cplx_out, accelerated);
  });
}

// FreeSpaceEvaluator::accumulate for one shift; outputs are read, added to, written back.
int ref_accumulate(void* p, size_t ns, const double* src, const double* charges, const double* forces,
                   const double* normals, const double* coeffs, size_t nt, const double* tgt, double shx,
                   double shy, int identity, int threads, int with_pressure, double* scalar, double* velocity,
                   double* pressure, double* cplx_io) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    ParticleSystem sys = system_of(ns, src, charges, forces, normals, coeffs, nt, tgt);
    ApplyOptions opt = options_of(1, threads, with_pressure, 0.0);
    FieldResult f = import_field(pz, nt, scalar, velocity, with_pressure ? pressure : nullptr, cplx_io);
    FreeSpaceEvaluator ev;
    ev.accumulate(pz, sys, Vec2{shx, shy}, identity != 0, opt, f);
    export_field(f, scalar, velocity, pressure, cplx_io, nullptr);
  });
}

int ref_choose_path(void* p, size_t ns, size_t nt) {
  return static_cast<int>(choose_path(*static_cast<Periodizer*>(p), ns, nt));
}

int ref_brute_force_far(void* p, int shells, size_t ns, const double* src, const double* charges,
                        const double* forces, const double* normals, const double* coeffs, size_t nt,
                        const double* tgt, int threads, double* scalar, double* velocity, double* cplx_out) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    ParticleSystem sys = system_of(ns, src, charges, forces, normals, coeffs, nt, tgt);
    FieldResult f = brute_force_far(pz, sys, shells, options_of(1, threads, 0, 0.0));
    export_field(f, scalar, velocity, nullptr, cplx_out, nullptr);
  });
}

int ref_periodicity_residual(void* p, int samples, size_t ns, const double* src, const double* charges,
                             const double* forces, const double* normals, const double* coeffs, int path,
                             int threads, double* e1, double* e2, double* scale) {
  return guarded([&] {
    const Periodizer& pz = *static_cast<Periodizer*>(p);
    ParticleSystem sys = system_of(ns, src, charges, forces, normals, coeffs, 0, nullptr);
    ResidualReport r = periodicity_residual(pz, sys, samples, options_of(path, threads, 0, 0.0));
    *e1 = r.e1;
    *e2 = r.e2;
    *scale = r.scale;
  });
}

// ---- NUFFT (backend 0 Reference, 1 Accelerated) ----
int ref_nufft_type1(int backend, double eps, size_t n, const double* x, const double* c, size_t nmodes, double* f) {
  return guarded([&] {
    std::vector<double> xv(x, x + n);
    std::vector<cplx> cv(n), fv;
    for (size_t i = 0; i < n; ++i) cv[i] = {c[2 * i], c[2 * i + 1]};
    nufft_type1(backend ? NufftBackend::Accelerated : NufftBackend::Reference, eps, xv, cv, nmodes, fv);
    put_cplx(fv, f);
  });
}

int ref_nufft_type2(int backend, double eps, size_t n, const double* x, size_t nmodes, const double* f, double* c) {
  return guarded([&] {
    std::vector<double> xv(x, x + n);
    std::vector<cplx> fv(nmodes), cv;
    for (size_t i = 0; i < nmodes; ++i) fv[i] = {f[2 * i], f[2 * i + 1]};
    nufft_type2(backend ? NufftBackend::Accelerated : NufftBackend::Reference, eps, xv, fv, cv);
    put_cplx(cv, c);
  });
}

int ref_nufft_type3(int backend, double eps, size_t n, const double* x, const double* c, size_t nk, const double* s,
                    double* f) {
  return guarded([&] {
    std::vector<double> xv(x, x + n), sv(s, s + nk);
    std::vector<cplx> cv(n), fv;
    for (size_t i = 0; i < n; ++i) cv[i] = {c[2 * i], c[2 * i + 1]};
    nufft_type3(backend ? NufftBackend::Accelerated : NufftBackend::Reference, eps, xv, cv, sv, fv);
    put_cplx(fv, f);
  });
}

// ---- kernels ----
int ref_bessel_kn(int l, double x, double* out) { return guarded([&] { *out = bessel_kn(l, x); }); }

int ref_greens_scalar(int pde, double beta, double rx, double ry, double* out) {
  return guarded([&] { *out = greens_scalar(static_cast<Pde>(pde), beta, {rx, ry}); });
}

int ref_greens_block(int pde, double beta, double rx, double ry, double* out) {
  return guarded([&] {
    Mat2 g = greens_block(static_cast<Pde>(pde), beta, {rx, ry});
    out[0] = g.a11;
    out[1] = g.a12;
    out[2] = g.a21;
    out[3] = g.a22;
  });
}

int ref_multipole_kernel(int pde, double beta, int l, double rx, double ry, double* out) {
  return guarded([&] {
    cplx v = multipole_kernel(static_cast<Pde>(pde), beta, l, {rx, ry});
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int ref_stresslet_dlp(double rx, double ry, double nx, double ny, double* out) {
  return guarded([&] {
    Mat2 g = stresslet_dlp({rx, ry}, {nx, ny});
    out[0] = g.a11;
    out[1] = g.a12;
    out[2] = g.a21;
    out[3] = g.a22;
  });
}

int ref_pressurelet(double rx, double ry, double* out) {
  return guarded([&] {
    Vec2 v = pressurelet({rx, ry});
    out[0] = v.x;
    out[1] = v.y;
  });
}

// ---- quadrature / truncation ----
int ref_truncation_order(double d, double xi, double eta, int periodicity, double eps, int* out) {
  return guarded([&] { *out = truncation_order(cell_of(d, xi, eta, periodicity), eps); });
}

int ref_gauss_legendre(int n, double* nodes, double* weights) {
  return guarded([&] {
    GaussRule g = gauss_legendre(n);
    for (int i = 0; i < n; ++i) {
      nodes[i] = g.nodes[i];
      weights[i] = g.weights[i];
    }
  });
}

int ref_sommerfeld_rule(int pde, double beta, double d, double xi, double eta, int periodicity, double eps,
                        double min_upper, size_t cap, double* nodes, double* weights, size_t* count, double* upper,
                        double* cert) {
  return guarded([&] {
    UnitCell cell = cell_of(d, xi, eta, periodicity);
    QuadratureRule r = sommerfeld_rule(static_cast<Pde>(pde), beta, cell, eps, min_upper);
    *count = r.size();
    *upper = r.upper;
    *cert = certify_rule(r, static_cast<Pde>(pde), beta, cell, eps);
    for (size_t i = 0; i < r.size() && i < cap; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
  });
}

int ref_interp_coeffs(double lo, double hi, int m, double x, double* out) {
  return guarded([&] {
    BarycentricGrid g = make_barycentric_grid(lo, hi, m);
    std::vector<double> c = interp_coeffs(g, x);
    for (int k = 0; k < m; ++k) out[k] = c[k];
  });
}

}  // extern "C"
