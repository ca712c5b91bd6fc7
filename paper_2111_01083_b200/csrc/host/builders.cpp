// Host periodizer builders: the plane-wave mode and coefficient tables the
// device plan uploads. O(rank) setup, once per (kernel, cell, eps).
// Restates /root/reference/proj/src/periodize_scalar.cpp,
// periodize_stokes.cpp, periodize_multipole.cpp and periodize_common.hpp
// (file:line per function); the math is PAPER.md:879-990 (south theorem and
// tail bound) and PAPER.md:1947-2000 (Stokes blocks).
#include <algorithm>
#include <cmath>
#include <utility>

#include "periwave/periwave.hpp"

namespace periwave {
namespace {

constexpr cplx kJ{0.0, 1.0};
constexpr double kSmallBeta = 1e-6;  // periodize_common.hpp:14

// e^{comp - 2Q} / (1 - e^{-Q}), Re Q > 0 (periodize_common.hpp:18-22).
cplx image_tail(cplx Q, double comp) { return std::exp(comp - 2.0 * Q) / (-cexpm1_neg(Q)); }

// (2 - e^{-Q}) / (1 - e^{-Q}) (periodize_common.hpp:26-29).
cplx weighted_tail_ratio(cplx Q) {
  const cplx e = std::exp(-Q);
  return (2.0 - e) / (1.0 - e);
}

// ((m0+1) - m0 e^{-x}) / (1 - e^{-x}) (periodize_common.hpp:33-36).
cplx weighted_tail_ratio_h(double x, int m0) {
  const double e = std::exp(-x);
  return cplx(((m0 + 1) - m0 * e) / (1.0 - e), 0.0);
}

// sum_{n in rows} e^{-m0 chi d + sgn n chi xi - i n lam eta} / (1 - e^{-chi d})
// (periodize_common.hpp:42-49).
cplx row_tail(const UnitCell& cell, double chi, double lam, double sgn) {
  const int nmax = cell.periodicity == Periodicity::Doubly ? 1 : 0;
  cplx s{0.0, 0.0};
  for (int n = -nmax; n <= nmax; ++n)
    s += std::exp(cplx(-cell.m0 * chi * cell.d + sgn * n * chi * cell.xi, -n * lam * cell.eta));
  return s / (-cexpm1_neg(cplx(chi * cell.d, 0.0)));
}

// Mode layout of periodize_common.hpp:60-82: south/west modes decay toward the
// far side, shifts put every stored exponent <= 0 on the rectangle.
void add_mode(ModeSet& ms, Axis axis, double half, double phase, double chi, bool first_side) {
  ms.axis = axis;
  ms.phase.push_back(phase);
  ms.decay_t.push_back(first_side ? -chi : chi);
  ms.decay_s.push_back(first_side ? chi : -chi);
  ms.shift_t.push_back(first_side ? -half : half);
  ms.shift_s.push_back(first_side ? half : -half);
}
void vertical_mode(ModeSet& ms, const UnitCell& c, double alpha, double chi, Direction dir) {
  add_mode(ms, Axis::Vertical, 0.5 * c.eta, alpha, chi, dir == Direction::South);
}
void horizontal_mode(ModeSet& ms, const UnitCell& c, double lam, double chi, Direction dir) {
  add_mode(ms, Axis::Horizontal, 0.5 * c.d, lam, chi, dir == Direction::West);
}

QuadratureRule checked_rule(Pde pde, double beta, const UnitCell& cell, double eps, double min_upper = 0.0) {
  QuadratureRule rule = sommerfeld_rule(pde, beta, cell, eps, min_upper);
  if (rule.size() == 0) return rule;
  require(certify_rule(rule, pde, beta, cell, eps) <= 100.0 * eps, ErrorCode::NotConverged,
          "half-line quadrature failed its self-check");
  return rule;
}

Mat2c conj_entries(const Mat2c& m) { return {std::conj(m.a11), std::conj(m.a12), std::conj(m.a21), std::conj(m.a22)}; }

// ------------------------------------------------------------- scalar kernels
// periodize_scalar.cpp:56-79
void scalar_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const bool screened = pz.pde == Pde::ModHelmholtz;
  const int M = truncation_order(c, pz.eps);
  for (Direction dir : {Direction::South, Direction::North}) {
    ScalarPart part;
    part.dir = dir;
    part.take_real = true;
    for (int m = -M; m <= M; ++m) {
      if (!screened && m == 0) continue;
      const double alpha = 2.0 * kPi * m / c.d;
      const double chi = screened ? std::hypot(alpha, pz.beta) : std::abs(alpha);
      cplx Q(chi * c.eta, -alpha * c.xi);
      if (dir == Direction::North) Q = std::conj(Q);
      vertical_mode(part.modes, c, alpha, chi, dir);
      part.diag.push_back(image_tail(Q, chi * c.eta) / (2.0 * c.d * chi));
    }
    if (!screened) {
      part.has_m0 = true;
      part.m0_coef = -1.0 / (2.0 * c.d * c.eta);
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// periodize_scalar.cpp:81-98
void scalar_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const bool screened = pz.pde == Pde::ModHelmholtz;
  for (Direction dir : {Direction::West, Direction::East}) {
    ScalarPart part;
    part.dir = dir;
    part.take_real = true;
    const double sgn = dir == Direction::West ? 1.0 : -1.0;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const double chi = screened ? std::hypot(lam, pz.beta) : lam;
      horizontal_mode(part.modes, c, lam, chi, dir);
      part.diag.push_back(rule.weights[k] / (2.0 * kPi * chi) * row_tail(c, chi, lam, sgn));
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// ------------------------------------------------------------- Stokes family
// periodize_stokes.cpp:19-25: extra vertical modes for symbols growing with chi.
int widened_order(const UnitCell& c, int base, double growth) {
  if (!(growth > 1.0)) return base;
  return base + static_cast<int>(std::ceil(c.d / (2.0 * kPi * c.eta) * std::log(growth)));
}

struct Rows {
  cplx sum{1.0, 0.0};
  cplx lin{0.0, 0.0};
};

// periodize_stokes.cpp:34-43
Rows rows_of(const UnitCell& c, double lam) {
  Rows r;
  if (c.periodicity == Periodicity::Doubly) {
    const cplx up = std::exp(cplx(lam * c.xi, -lam * c.eta));
    const cplx dn = std::exp(cplx(-lam * c.xi, lam * c.eta));
    r.sum += up + dn;
    r.lin = up - dn;
  }
  return r;
}

// periodize_stokes.cpp:45-71
void stokes_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const int base = truncation_order(c, pz.eps);
  const double chi0 = 2.0 * kPi * base / c.d;
  const int M = widened_order(c, base, chi0 * c.eta);
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    BlockPart part;
    part.dir = dir;
    part.three_term = true;
    for (int m = -M; m <= M; ++m) {
      if (m == 0) continue;
      const double alpha = 2.0 * kPi * m / c.d;
      const double a = std::abs(alpha);
      const double sg = (m > 0) == south ? 1.0 : -1.0;
      const cplx Q(a * c.eta, (south ? -alpha : alpha) * c.xi);
      const cplx t = image_tail(Q, a * c.eta) / (4.0 * c.d);
      const Mat2c sym{1.0, kJ * sg, kJ * sg, -1.0};
      vertical_mode(part.modes, c, alpha, a, dir);
      part.diag_a.push_back((eye * (1.0 / a) + sym * (-weighted_tail_ratio(Q) * c.eta)) * t);
      part.diag_b.push_back(sym * (south ? t : -t));
    }
    part.has_m0 = true;
    part.m0_mat = {-1.0 / (2.0 * c.d * c.eta), 0.0, 0.0, 0.0};
    pz.block_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:73-100
void stokes_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  const Mat2c wsym{-1.0, kJ, kJ, 1.0};
  for (Direction dir : {Direction::West, Direction::East}) {
    const bool west = dir == Direction::West;
    BlockPart part;
    part.dir = dir;
    part.three_term = true;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const Rows rb = rows_of(c, lam);
      const double t0 = std::exp(-c.m0 * lam * c.d) / (-std::expm1(-lam * c.d));
      const cplx g = weighted_tail_ratio_h(lam * c.d, c.m0);
      const double amp = rule.weights[k] * t0 / (4.0 * kPi);
      Mat2c da = (eye * (rb.sum / lam) + wsym * (-(g * c.d * rb.sum - c.xi * rb.lin))) * amp;
      Mat2c db = wsym * (amp * rb.sum);
      if (!west) {
        da = conj_entries(da);
        db = conj_entries(db) * cplx(-1.0);
      }
      horizontal_mode(part.modes, c, lam, lam, dir);
      part.diag_a.push_back(da);
      part.diag_b.push_back(db);
    }
    pz.block_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:102-139
void mod_stokes_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const double b2 = pz.beta * pz.beta;
  const int base = truncation_order(c, pz.eps);
  const double chi0 = 2.0 * kPi * base / c.d;
  const int M = widened_order(c, base, std::max(chi0 * chi0 / b2, chi0 * c.eta));
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    const double sx = south ? -1.0 : 1.0;
    const double si = south ? 1.0 : -1.0;
    BlockPart part;
    part.dir = dir;
    for (int m = -M; m <= M; ++m) {  // screened family, m = 0 included
      const double alpha = 2.0 * kPi * m / c.d;
      const double chi = std::hypot(alpha, pz.beta);
      const cplx Q(chi * c.eta, sx * alpha * c.xi);
      const cplx t = image_tail(Q, chi * c.eta) / (2.0 * b2 * c.d);
      const cplx ia = kJ * (si * alpha);
      vertical_mode(part.modes, c, alpha, chi, dir);
      part.diag_a.push_back({chi * t, ia * t, ia * t, -(alpha * alpha / chi) * t});
    }
    for (int m = -M; m <= M; ++m) {  // unscreened companion, m = 0 symbol vanishes
      if (m == 0) continue;
      const double alpha = 2.0 * kPi * m / c.d;
      const double a = std::abs(alpha);
      const cplx Q(a * c.eta, sx * alpha * c.xi);
      const cplx t = image_tail(Q, a * c.eta) / (2.0 * b2 * c.d);
      const cplx ia = kJ * (si * alpha);
      vertical_mode(part.modes, c, alpha, a, dir);
      part.diag_a.push_back({-a * t, -ia * t, -ia * t, a * t});
    }
    pz.block_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:141-164
void mod_stokes_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const double b2 = pz.beta * pz.beta;
  for (Direction dir : {Direction::West, Direction::East}) {
    const double sgn = dir == Direction::West ? 1.0 : -1.0;
    BlockPart part;
    part.dir = dir;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const double chi = std::hypot(lam, pz.beta);
      const cplx il = kJ * (sgn * lam);
      const cplx tb = row_tail(c, chi, lam, sgn) * (rule.weights[k] / (2.0 * kPi * b2));
      horizontal_mode(part.modes, c, lam, chi, dir);
      part.diag_a.push_back({-(lam * lam / chi) * tb, il * tb, il * tb, chi * tb});
      const cplx tz = row_tail(c, lam, lam, sgn) * (rule.weights[k] / (2.0 * kPi * b2));
      horizontal_mode(part.modes, c, lam, lam, dir);
      part.diag_a.push_back({lam * tz, -il * tz, -il * tz, -lam * tz});
    }
    pz.block_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:166-189
void pressure_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const int base = truncation_order(c, pz.eps);
  const double chi0 = 2.0 * kPi * base / c.d;
  const int M = widened_order(c, base, chi0 * c.eta);
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    PressurePart part;
    part.dir = dir;
    for (int m = -M; m <= M; ++m) {
      if (m == 0) continue;
      const double alpha = 2.0 * kPi * m / c.d;
      const double a = std::abs(alpha);
      const cplx Q(a * c.eta, (south ? -alpha : alpha) * c.xi);
      vertical_mode(part.modes, c, alpha, a, dir);
      part.diag.push_back(-image_tail(Q, a * c.eta) / (2.0 * c.d * a));
      part.row.push_back({kJ * alpha, cplx(south ? -a : a)});
    }
    part.has_m0 = true;
    part.m0_coef = 1.0 / (2.0 * c.d * c.eta);
    part.m0_row = {0.0, 1.0};
    pz.pressure_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:191-207
void pressure_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  for (Direction dir : {Direction::West, Direction::East}) {
    const double sgn = dir == Direction::West ? 1.0 : -1.0;
    PressurePart part;
    part.dir = dir;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      horizontal_mode(part.modes, c, lam, lam, dir);
      part.diag.push_back(row_tail(c, lam, lam, sgn) * (rule.weights[k] / (2.0 * kPi * lam)));
      part.row.push_back({cplx(sgn * lam), -kJ * lam});
    }
    pz.pressure_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:209-246
void dlp_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const int base = truncation_order(c, pz.eps);
  const double chi0 = 2.0 * kPi * base / c.d;
  const int M = widened_order(c, base, chi0 * c.eta * chi0 * c.eta);
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    StressletPart part;
    part.dir = dir;
    for (int m = -M; m <= M; ++m) {
      if (m == 0) continue;
      const double alpha = 2.0 * kPi * m / c.d;
      const double a = std::abs(alpha);
      const double sg = m > 0 ? 1.0 : -1.0;
      const cplx Q(a * c.eta, (south ? -alpha : alpha) * c.xi);
      const cplx amp = image_tail(Q, a * c.eta) / (2.0 * c.d);
      vertical_mode(part.modes, c, alpha, a, dir);
      const double sside = south ? 1.0 : -1.0;
      part.a1.push_back(Mat2c{2.0 * kJ * sg, -sside, -sside, 0.0} * amp);
      part.a2.push_back(eye * (-sside * amp));
      part.sa.push_back(kJ * alpha);
      part.sb.push_back(cplx(-sside * a));
      part.smat.push_back(Mat2c{sside, kJ * sg, kJ * sg, -sside} * (-amp));
      part.off.push_back(sside * weighted_tail_ratio(Q) * c.eta);
    }
    part.has_m0 = true;
    part.m0_coef = 1.0 / (2.0 * c.d * c.eta);
    pz.stresslet_parts.push_back(std::move(part));
  }
}

// periodize_stokes.cpp:248-277
void dlp_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  for (Direction dir : {Direction::West, Direction::East}) {
    const bool west = dir == Direction::West;
    StressletPart part;
    part.dir = dir;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const Rows rb = rows_of(c, lam);
      const cplx bb = west ? rb.sum : std::conj(rb.sum);
      const cplx bp = west ? rb.lin : -std::conj(rb.lin);
      const double t0 = std::exp(-c.m0 * lam * c.d) / (-std::expm1(-lam * c.d));
      const cplx g = weighted_tail_ratio_h(lam * c.d, c.m0);
      const double amp0 = rule.weights[k] * t0 / (2.0 * kPi);
      const Mat2c m1 = west ? eye * cplx(-1.0) : eye;
      const Mat2c m2 = west ? Mat2c{0.0, -1.0, -1.0, 2.0 * kJ} : Mat2c{0.0, 1.0, 1.0, 2.0 * kJ};
      const cplx sa = west ? cplx(-lam) : cplx(lam);
      const cplx sb = kJ * lam;
      const Mat2c cm = west ? Mat2c{-1.0, kJ, kJ, 1.0} : Mat2c{1.0, kJ, kJ, -1.0};
      horizontal_mode(part.modes, c, lam, lam, dir);
      part.a1.push_back((m1 * bb + cm * (c.xi * sa * bp)) * amp0);
      part.a2.push_back((m2 * bb + cm * (c.xi * sb * bp)) * amp0);
      part.sa.push_back(sa);
      part.sb.push_back(sb);
      part.smat.push_back(cm * (-amp0 * bb));
      part.off.push_back((west ? g : -g) * c.d);
    }
    pz.stresslet_parts.push_back(std::move(part));
  }
}

// ------------------------------------------------------------- multipole sources
cplx cpow_int(cplx z, int l) {
  cplx r{1.0, 0.0};
  for (int i = 0; i < l; ++i) r *= z;
  return r;
}
double factorial_small(int n) { return n <= 1 ? 1.0 : n == 2 ? 2.0 : 6.0; }

// periodize_multipole.cpp:29-37: keep extending past base and the symbol peak
// until the mode magnitude drops below cutoff * running max.
struct Extension {
  int base = 0, peak = 0;
  double cutoff = 0.0, dmax = 0.0;
  bool stop(int mabs, double mag) const { return mabs > std::max(base, peak) && mag <= cutoff * dmax; }
};
constexpr int kMaxModes = 10000000;

// periodize_multipole.cpp:39-79
void mh_multipole_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const int l = pz.multipole_order;
  const double beta = pz.beta;
  const int base = truncation_order(c, pz.eps);
  const int peak = static_cast<int>(std::ceil(l * c.d / (2.0 * kPi * c.eta))) + 1;
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    const cplx pref = cpow_int(south ? kJ : -kJ, l) * (kPi / c.d);
    ScalarPart part;
    part.dir = dir;
    part.take_real = false;
    Extension ext{base, peak, 0.1 * pz.eps, 0.0};
    auto push = [&](int m) {
      const double alpha = 2.0 * kPi * m / c.d;
      const double chi = std::hypot(alpha, beta);
      double ratio;
      if (south)
        ratio = alpha >= 0.0 ? beta / (chi + alpha) : (chi - alpha) / beta;
      else
        ratio = alpha >= 0.0 ? (chi + alpha) / beta : beta / (chi - alpha);
      const cplx Q(chi * c.eta, (south ? -alpha : alpha) * c.xi);
      const cplx dv = pref * (std::pow(ratio, l) / chi) * image_tail(Q, chi * c.eta);
      const double mag = std::abs(dv);
      if (ext.stop(std::abs(m), mag)) return false;
      ext.dmax = std::max(ext.dmax, mag);
      vertical_mode(part.modes, c, alpha, chi, dir);
      part.diag.push_back(dv);
      return true;
    };
    for (int m = -base; m <= base; ++m) push(m);
    const int step = south ? -1 : 1;
    for (int m = step * (base + 1);; m += step) {
      require(std::abs(m) < kMaxModes, ErrorCode::NotConverged, "multipole vertical mode extension did not terminate");
      if (!push(m)) break;
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// periodize_multipole.cpp:81-116
void laplace_multipole_vertical(Periodizer& pz) {
  const UnitCell& c = pz.cell;
  const int l = pz.multipole_order;
  const int base = truncation_order(c, pz.eps);
  const int peak = static_cast<int>(std::ceil((l - 1) * c.d / (2.0 * kPi * c.eta))) + 1;
  for (Direction dir : {Direction::South, Direction::North}) {
    const bool south = dir == Direction::South;
    const cplx c0 = cpow_int((south ? -kJ : kJ) * (2.0 * kPi / c.d), l) / factorial_small(l - 1);
    ScalarPart part;
    part.dir = dir;
    part.take_real = false;
    Extension ext{base, peak, 0.1 * pz.eps, 0.0};
    auto push = [&](int m) {
      const double alpha = 2.0 * kPi * m / c.d;
      const cplx Q(alpha * c.eta, -alpha * c.xi);
      const cplx dv = c0 * std::pow(static_cast<double>(m), l - 1) * image_tail(Q, alpha * c.eta);
      const double mag = std::abs(dv);
      if (ext.stop(m, mag)) return false;
      ext.dmax = std::max(ext.dmax, mag);
      vertical_mode(part.modes, c, south ? alpha : -alpha, alpha, dir);
      part.diag.push_back(dv);
      return true;
    };
    for (int m = 1; m <= base; ++m) push(m);
    for (int m = base + 1;; ++m) {
      require(m < kMaxModes, ErrorCode::NotConverged, "multipole vertical mode extension did not terminate");
      if (!push(m)) break;
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// periodize_multipole.cpp:118-144
void mh_multipole_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const int l = pz.multipole_order;
  const double beta = pz.beta;
  for (Direction dir : {Direction::West, Direction::East}) {
    const bool west = dir == Direction::West;
    const double sdir = west ? 1.0 : -1.0;
    const cplx pref = (west || l % 2 == 0 ? 1.0 : -1.0) / (2.0 * std::pow(beta, l));
    ScalarPart part;
    part.dir = dir;
    part.take_real = false;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const double chi = std::hypot(lam, beta);
      for (double lt : {lam, -lam}) {
        const double symbol = sdir * lt >= 0.0 ? chi + sdir * lt : beta * beta / (chi + std::abs(lt));
        horizontal_mode(part.modes, c, lt, chi, dir);
        part.diag.push_back(pref * std::pow(symbol, l) * (rule.weights[k] / chi) * row_tail(c, chi, lt, sdir));
      }
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// periodize_multipole.cpp:146-169
void laplace_multipole_horizontal(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const int l = pz.multipole_order;
  const bool doubly = c.periodicity == Periodicity::Doubly;
  for (Direction dir : {Direction::West, Direction::East}) {
    const bool west = dir == Direction::West;
    const double pref = (west || l % 2 == 0) ? 1.0 : -1.0;
    ScalarPart part;
    part.dir = dir;
    part.take_real = false;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      cplx br{1.0, 0.0};
      if (doubly) br += std::exp(cplx(lam * c.xi, lam * c.eta)) + std::exp(cplx(-lam * c.xi, -lam * c.eta));
      const double t0 = std::exp(-c.m0 * lam * c.d) / (-std::expm1(-lam * c.d));
      horizontal_mode(part.modes, c, west ? -lam : lam, lam, dir);
      part.diag.push_back(pref * std::pow(lam, l - 1) / factorial_small(l - 1) * rule.weights[k] * br * t0);
    }
    pz.scalar_parts.push_back(std::move(part));
  }
}

// periodize_multipole.cpp:174-203: extend the half-line truncation until the
// growing multipole symbol has fallen a full eps below its peak.
double multipole_truncation(Pde pde, double beta, int l, const UnitCell& c, double eps) {
  const double gap = c.m0 * c.d - std::abs(c.xi);
  const double eta_osc = c.periodicity == Periodicity::Doubly ? 2.0 * c.eta : c.eta;
  const double lam0 = 2.0 * kPi / eta_osc;
  auto logmag = [&](double lam) {
    if (pde == Pde::ModHelmholtz) {
      const double chi = std::hypot(lam, beta);
      return l * std::log((chi + lam) / beta) - chi * gap - std::log(chi) - std::log(-std::expm1(-chi * c.d));
    }
    return (l - 1) * std::log(lam) - lam * gap - std::log(-std::expm1(-lam * c.d));
  };
  const QuadratureRule plain = sommerfeld_rule(pde, beta, c, eps);
  const double up0 = plain.upper > 0.0 ? plain.upper : std::log(1.0 / eps) / c.d;
  const double lo = 1e-2 * lam0;
  const double hi = std::max(up0, 4.0 * lam0);
  double peak = -1e300;
  for (int i = 0; i < 400; ++i) peak = std::max(peak, logmag(lo * std::pow(hi / lo, i / 399.0)));
  const double cut = peak + std::log(0.1 * eps);
  double up = std::max(up0, lam0);
  int guard = 0;
  while (logmag(up) > cut) {
    up += 0.5 * lam0;
    require(++guard < 2000000, ErrorCode::NotConverged, "multipole truncation scan did not terminate");
  }
  return up;
}

void check_eps(double eps) {
  require(eps >= 1e-14 && eps < 0.1, ErrorCode::PrecisionOutOfRange, "eps must lie in [1e-14, 0.1)");
}

}  // namespace

// periodize_scalar.cpp:11-18 (Theorem 3.1)
int truncation_order(const UnitCell& cell, double eps) {
  check_eps(eps);
  const double x = 2.0 * kPi * cell.eta / cell.d;
  const double m = cell.d / (2.0 * kPi * cell.eta) * std::log(1.0 / (-std::expm1(-x) * eps));
  return static_cast<int>(std::ceil(m));
}

// periodize_scalar.cpp:20-26
double vertical_tail_bound(const UnitCell& cell, int M) {
  require(M >= 1, ErrorCode::InvalidOrder, "tail bound needs M >= 1");
  const double t = 2.0 * kPi * (M + 1) * cell.eta / cell.d;
  const double t1 = 2.0 * kPi * cell.eta / cell.d;
  return std::exp(-t) / (2.0 * kPi * (M + 1) * (-std::expm1(-t)) * (-std::expm1(-t1)));
}

std::size_t Periodizer::rank() const {
  std::size_t r = 0;
  for (const auto& p : scalar_parts) r += p.modes.size();
  for (const auto& p : block_parts) r += p.modes.size();
  for (const auto& p : pressure_parts) r += p.modes.size();
  for (const auto& p : stresslet_parts) r += p.modes.size();
  return r;
}

// periodize_scalar.cpp:102-136
Periodizer make_periodizer(Pde pde, double beta, const UnitCell& cell, double eps) {
  check_eps(eps);
  const bool screened = pde == Pde::ModHelmholtz || pde == Pde::ModStokes;
  if (screened) require(beta > 0.0, ErrorCode::MissingBeta, "screened kernel needs beta > 0");
  Periodizer pz;
  pz.pde = pde;
  pz.beta = screened ? beta : 0.0;
  pz.cell = cell;
  pz.eps = eps;
  pz.requires_neutrality = screened ? (beta < kSmallBeta) : true;
  const bool doubly = cell.periodicity == Periodicity::Doubly;
  switch (pde) {
    case Pde::Poisson:
    case Pde::ModHelmholtz:
      if (doubly) scalar_vertical(pz);
      scalar_horizontal(pz, checked_rule(pde, pz.beta, cell, eps));
      break;
    case Pde::Stokes: {
      if (doubly) stokes_vertical(pz);
      const QuadratureRule rule = checked_rule(Pde::Stokes, 0.0, cell, eps);
      stokes_horizontal(pz, rule);
      if (doubly) pressure_vertical(pz);
      pressure_horizontal(pz, rule);
      break;
    }
    case Pde::ModStokes: {
      if (doubly) mod_stokes_vertical(pz);
      const QuadratureRule rule = checked_rule(Pde::Stokes, 0.0, cell, eps);
      mod_stokes_horizontal(pz, rule);
      if (doubly) pressure_vertical(pz);
      pressure_horizontal(pz, rule);
      break;
    }
  }
  return pz;
}

// periodize_stokes.cpp:302-315
Periodizer make_stokes_dlp_periodizer(const UnitCell& cell, double eps) {
  check_eps(eps);
  Periodizer pz;
  pz.pde = Pde::Stokes;
  pz.cell = cell;
  pz.eps = eps;
  pz.dlp = true;
  pz.requires_neutrality = true;
  if (cell.periodicity == Periodicity::Doubly) dlp_vertical(pz);
  dlp_horizontal(pz, checked_rule(Pde::Stokes, 0.0, cell, eps));
  return pz;
}

// periodize_multipole.cpp:207-239
Periodizer make_multipole_periodizer(Pde pde, double beta, int l, const UnitCell& cell, double eps) {
  check_eps(eps);
  require(pde == Pde::Poisson || pde == Pde::ModHelmholtz, ErrorCode::Unsupported,
          "multipole periodizers cover the scalar kernels only");
  require(l >= 1 && l <= 4, ErrorCode::OrderOutOfRange, "multipole order must lie in 1..4");
  const bool screened = pde == Pde::ModHelmholtz;
  if (screened) require(beta > 0.0, ErrorCode::MissingBeta, "screened kernel needs beta > 0");
  Periodizer pz;
  pz.pde = pde;
  pz.beta = screened ? beta : 0.0;
  pz.cell = cell;
  pz.eps = eps;
  pz.multipole_order = l;
  pz.requires_neutrality = pde == Pde::Poisson && l == 1;
  const double up = multipole_truncation(pde, pz.beta, l, cell, eps);
  const QuadratureRule rule = checked_rule(pde, pz.beta, cell, eps, up);
  if (cell.periodicity == Periodicity::Doubly) {
    if (screened)
      mh_multipole_vertical(pz);
    else
      laplace_multipole_vertical(pz);
  }
  if (screened)
    mh_multipole_horizontal(pz, rule);
  else
    laplace_multipole_horizontal(pz, rule);
  return pz;
}

}  // namespace periwave
