// Plane-wave tables of the periodizers (host, O(rank), once per kernel / cell / eps): the
// mode sets and diagonal coefficients the device plan uploads (engine.cu build_families).
//
// Geometry. The lattice images outside the near 3 x 3 (or 3 x 1) block fall into four
// strips: south / north of the cell (vertical strips, periodic in x with period d) and
// west / east of it (horizontal strips, an integral over the spectral variable lambda).
// Every strip contributes sum_r T_l(r) diag_r sum_j S_j(r) q_j with the separable mode
// factors of PAPER.md:879-990:
//     S_j(r) = e^{decay_s (w_j - shift_s)} e^{-i phase p_j},  T_l(r) = e^{decay_t (w_l - shift_t)} e^{+i phase p_l}
// (w the decay coordinate: y on the vertical strips, x on the horizontal ones; p the other
// one). The decay always points away from the strip, and the shifts put every stored
// exponent at or below zero on the rectangle (Strip::place).
//
// Vertical strips: Fourier modes alpha_m = 2 pi m / d, |m| <= M (truncation_order). A
// strip's image rows n >= 2 (south) sum geometrically: with Q = chi eta -+ i alpha xi the
// south theorem gives the tail e^{-2Q} / (1 - e^{-Q}) (the e^{chi eta} in strip_tail undoes
// the two shifts). Horizontal strips: the half-line rule's nodes lambda_k with weights
// w_k (quad_rules.cpp); image columns |m| > m0 sum to e^{-m0 chi d} / (1 - e^{-chi d}), the
// three (doubly periodic) or one (singly) image rows add e^{+-chi xi -+ i lambda eta}.
//
// Per kernel the diagonal is the strip symbol of its Green's function:
//   Laplace / modified Helmholtz  1 / (2 chi) [per d] or w / (2 pi chi)
//   Stokes (three-term blocks)
//   modified Stokes               difference of the screened and unscreened symbols over beta^2
//   pressure, stresslet (DLP), multipole sources: their own symbols below.
// The tables match the reference's (tests/test_builders.py, within 1e-15) so the near /
// far split and every rank are the reference's; interfaces /root/reference/proj/include/
// periwave/periodize.hpp:12-130.
#include <algorithm>
#include <cmath>
#include <functional>
#include <utility>

#include "periwave/periwave.hpp"

namespace periwave {
namespace {

constexpr cplx kI{0.0, 1.0};
constexpr double kUnscreenedBeta = 1e-6;  // a "screened" kernel this weak needs neutral data
constexpr int kModeCap = 10000000;         // runaway guard of the multipole mode extension

void require_eps(double eps) {
  require(eps >= 1e-14 && eps < 0.1, ErrorCode::PrecisionOutOfRange, "precision must lie in [1e-14, 0.1)");
}

// ---------------------------------------------------------------- strips
struct Strip {
  Direction dir;
  Axis axis;
  bool lower;   // south / west: the strip lies below / left of the cell
  double half;  // eta / 2 (vertical) or d / 2 (horizontal)

  static Strip of(const UnitCell& c, Direction d) {
    const bool vertical = d == Direction::South || d == Direction::North;
    return {d, vertical ? Axis::Vertical : Axis::Horizontal, d == Direction::South || d == Direction::West,
            vertical ? 0.5 * c.eta : 0.5 * c.d};
  }
  double side() const { return lower ? 1.0 : -1.0; }

  // one mode: targets decay toward the strip, sources away from it
  void place(ModeSet& ms, double phase, double chi) const {
    ms.axis = axis;
    ms.phase.push_back(phase);
    ms.decay_t.push_back(lower ? -chi : chi);
    ms.decay_s.push_back(lower ? chi : -chi);
    ms.shift_t.push_back(lower ? -half : half);
    ms.shift_s.push_back(lower ? half : -half);
  }
};

// (a strip without modes keeps ModeSet's default axis, as the reference's tables do)
template <class Part>
Part part_on(const Strip& s) {
  Part p;
  p.dir = s.dir;
  return p;
}

// e^{comp - 2Q} / (1 - e^{-Q}), Re Q > 0: the geometric sum over a vertical strip's image
// rows, comp = chi eta compensating the two stored shifts.
cplx strip_tail(cplx Q, double comp) { return std::exp(comp - 2.0 * Q) / (-cexpm1_neg(Q)); }

// Q of a vertical strip for decay chi and phase alpha: chi eta - i alpha xi (south),
// its conjugate (north).
cplx strip_q(const UnitCell& c, const Strip& s, double chi, double alpha) {
  return {chi * c.eta, (s.lower ? -alpha : alpha) * c.xi};
}

// sum_{rows n} e^{-m0 chi d + side n chi xi - i n lambda eta} / (1 - e^{-chi d}): the image
// columns beyond m0 and the image rows of a horizontal strip.
cplx column_tail(const UnitCell& c, double chi, double lam, double side) {
  const int rows = c.periodicity == Periodicity::Doubly ? 1 : 0;
  cplx acc{0.0, 0.0};
  for (int n = -rows; n <= rows; ++n) acc += std::exp(cplx(-c.m0 * chi * c.d + side * n * chi * c.xi, -n * lam * c.eta));
  return acc / (-cexpm1_neg(cplx(chi * c.d, 0.0)));
}

// e^{-m0 lambda d} / (1 - e^{-lambda d}) (the unscreened column tail without rows)
double column_tail_plain(const UnitCell& c, double lam) { return std::exp(-c.m0 * lam * c.d) / (-std::expm1(-lam * c.d)); }

// image rows of a horizontal strip for the block kernels: 1 (+ e^{lambda xi - i lambda eta}
// + e^{-lambda xi + i lambda eta} when doubly periodic) and the odd combination
struct RowSums {
  cplx even{1.0, 0.0};
  cplx odd{0.0, 0.0};
};
RowSums row_sums(const UnitCell& c, double lam) {
  RowSums r;
  if (c.periodicity == Periodicity::Doubly) {
    const cplx up = std::exp(cplx(lam * c.xi, -lam * c.eta)), down = std::exp(cplx(-lam * c.xi, lam * c.eta));
    r.even += up + down;
    r.odd = up - down;
  }
  return r;
}

// (2 - e^{-Q}) / (1 - e^{-Q}) and ((m0 + 1) - m0 e^{-x}) / (1 - e^{-x}): the first
// moments of the image-row / image-column tails (the three-term blocks' linear terms)
cplx tail_moment(cplx Q) {
  const cplx e = std::exp(-Q);
  return (2.0 - e) / (1.0 - e);
}
cplx tail_moment_columns(double x, int m0) {
  const double e = std::exp(-x);
  return cplx(((m0 + 1) - m0 * e) / (1.0 - e), 0.0);
}

Mat2c conj(const Mat2c& m) { return {std::conj(m.a11), std::conj(m.a12), std::conj(m.a21), std::conj(m.a22)}; }

// Fourier modes -M..M of a vertical strip (m = 0 optional)
void each_fourier(const UnitCell& c, int M, bool with_zero, const std::function<void(int, double)>& fn) {
  for (int m = -M; m <= M; ++m)
    if (with_zero || m != 0) fn(m, 2.0 * kPi * m / c.d);
}

// more vertical modes for symbols that grow with chi: the tail bound's decay e^{-chi eta}
// has to absorb the growth (periodize_stokes.cpp:19-25)
int widen(const UnitCell& c, int base, double growth) {
  if (!(growth > 1.0)) return base;
  return base + static_cast<int>(std::ceil(c.d / (2.0 * kPi * c.eta) * std::log(growth)));
}

QuadratureRule certified_rule(Pde pde, double beta, const UnitCell& cell, double eps, double min_upper = 0.0) {
  QuadratureRule r = sommerfeld_rule(pde, beta, cell, eps, min_upper);
  if (r.size())
    require(certify_rule(r, pde, beta, cell, eps) <= 100.0 * eps, ErrorCode::NotConverged,
            "the lambda rule does not reach the requested precision");
  return r;
}

constexpr Direction kVertical[] = {Direction::South, Direction::North};
constexpr Direction kHorizontal[] = {Direction::West, Direction::East};

// ---------------------------------------------------------------- scalar kernels
// Laplace (chi = |alpha|, m = 0 handled by the rank-one term -y y' / (2 d eta)) and the
// modified Helmholtz kernel (chi = sqrt(alpha^2 + beta^2), m = 0 included).
void scalar_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const bool screened = pz.pde == Pde::ModHelmholtz;
  auto chi_of = [&](double k) { return screened ? std::hypot(k, pz.beta) : std::abs(k); };
  if (c.periodicity == Periodicity::Doubly) {
    const int M = truncation_order(c, pz.eps);
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<ScalarPart>(s);
      p.take_real = true;
      each_fourier(c, M, screened, [&](int, double alpha) {
        const double chi = chi_of(alpha);
        s.place(p.modes, alpha, chi);
        p.diag.push_back(strip_tail(strip_q(c, s, chi, alpha), chi * c.eta) / (2.0 * c.d * chi));
      });
      if (!screened) {
        p.has_m0 = true;
        p.m0_coef = -1.0 / (2.0 * c.d * c.eta);
      }
      pz.scalar_parts.push_back(std::move(p));
    }
  }
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    auto p = part_on<ScalarPart>(s);
    p.take_real = true;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k], chi = chi_of(lam);
      s.place(p.modes, lam, chi);
      p.diag.push_back(rule.weights[k] / (2.0 * kPi * chi) * column_tail(c, chi, lam, s.side()));
    }
    pz.scalar_parts.push_back(std::move(p));
  }
}

// ---------------------------------------------------------------- Stokes velocity
// Three-term blocks: u += T (D_a s1 + D_b s2 - w_l D_b s1) with s2
// the y- (x-) weighted source sums; D_a carries the 1/chi identity part and the tail's
// first moment, D_b the symmetric rank-one symbol.
void stokes_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  if (c.periodicity == Periodicity::Doubly) {
    const int base = truncation_order(c, pz.eps);
    const int M = widen(c, base, 2.0 * kPi * base / c.d * c.eta);
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<BlockPart>(s);
      p.three_term = true;
      each_fourier(c, M, false, [&](int m, double alpha) {
        const double a = std::abs(alpha);
        const double sg = (m > 0) == s.lower ? 1.0 : -1.0;
        const cplx Q = strip_q(c, s, a, alpha);
        const cplx t = strip_tail(Q, a * c.eta) / (4.0 * c.d);
        const Mat2c sym{1.0, kI * sg, kI * sg, -1.0};
        s.place(p.modes, alpha, a);
        p.diag_a.push_back((eye * (1.0 / a) + sym * (-tail_moment(Q) * c.eta)) * t);
        p.diag_b.push_back(sym * (s.lower ? t : -t));
      });
      p.has_m0 = true;
      p.m0_mat = {-1.0 / (2.0 * c.d * c.eta), 0.0, 0.0, 0.0};
      pz.block_parts.push_back(std::move(p));
    }
  }
  const Mat2c wsym{-1.0, kI, kI, 1.0};
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    auto p = part_on<BlockPart>(s);
    p.three_term = true;
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const RowSums rows = row_sums(c, lam);
      const double amp = rule.weights[k] * column_tail_plain(c, lam) / (4.0 * kPi);
      Mat2c da = (eye * (rows.even / lam) +
                  wsym * (-(tail_moment_columns(lam * c.d, c.m0) * c.d * rows.even - c.xi * rows.odd))) *
                 amp;
      Mat2c db = wsym * (amp * rows.even);
      if (!s.lower) {  // east: the mirror image of west
        da = conj(da);
        db = conj(db) * cplx(-1.0);
      }
      s.place(p.modes, lam, lam);
      p.diag_a.push_back(da);
      p.diag_b.push_back(db);
    }
    pz.block_parts.push_back(std::move(p));
  }
}

// Modified Stokes: (screened symbol - unscreened symbol) / beta^2, one mode set per
// symbol on every strip (two-term blocks).
void mod_stokes_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const double b2 = pz.beta * pz.beta;
  if (c.periodicity == Periodicity::Doubly) {
    const int base = truncation_order(c, pz.eps);
    const double chi0 = 2.0 * kPi * base / c.d;
    const int M = widen(c, base, std::max(chi0 * chi0 / b2, chi0 * c.eta));
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<BlockPart>(s);
      each_fourier(c, M, true, [&](int, double alpha) {  // screened: chi = sqrt(alpha^2 + beta^2)
        const double chi = std::hypot(alpha, pz.beta);
        const cplx t = strip_tail(strip_q(c, s, chi, alpha), chi * c.eta) / (2.0 * b2 * c.d);
        const cplx ia = kI * (s.side() * alpha);
        s.place(p.modes, alpha, chi);
        p.diag_a.push_back({chi * t, ia * t, ia * t, -(alpha * alpha / chi) * t});
      });
      each_fourier(c, M, false, [&](int, double alpha) {  // unscreened companion
        const double a = std::abs(alpha);
        const cplx t = strip_tail(strip_q(c, s, a, alpha), a * c.eta) / (2.0 * b2 * c.d);
        const cplx ia = kI * (s.side() * alpha);
        s.place(p.modes, alpha, a);
        p.diag_a.push_back({-a * t, -ia * t, -ia * t, a * t});
      });
      pz.block_parts.push_back(std::move(p));
    }
  }
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    auto p = part_on<BlockPart>(s);
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k], chi = std::hypot(lam, pz.beta);
      const cplx il = kI * (s.side() * lam);
      const double wk = rule.weights[k] / (2.0 * kPi * b2);
      const cplx ts = column_tail(c, chi, lam, s.side()) * wk;
      s.place(p.modes, lam, chi);
      p.diag_a.push_back({-(lam * lam / chi) * ts, il * ts, il * ts, chi * ts});
      const cplx tu = column_tail(c, lam, lam, s.side()) * wk;
      s.place(p.modes, lam, lam);
      p.diag_a.push_back({lam * tu, -il * tu, -il * tu, -lam * tu});
    }
    pz.block_parts.push_back(std::move(p));
  }
}

// Pressure of the Stokes-family single layer: p = grad(log) . f / (2 pi) -> one row
// vector per mode (i alpha, -+|alpha|) and a rank-one y term.
void pressure_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  if (c.periodicity == Periodicity::Doubly) {
    const int base = truncation_order(c, pz.eps);
    const int M = widen(c, base, 2.0 * kPi * base / c.d * c.eta);
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<PressurePart>(s);
      each_fourier(c, M, false, [&](int, double alpha) {
        const double a = std::abs(alpha);
        s.place(p.modes, alpha, a);
        p.diag.push_back(-strip_tail(strip_q(c, s, a, alpha), a * c.eta) / (2.0 * c.d * a));
        p.row.push_back({kI * alpha, cplx(s.lower ? -a : a)});
      });
      p.has_m0 = true;
      p.m0_coef = 1.0 / (2.0 * c.d * c.eta);
      p.m0_row = {0.0, 1.0};
      pz.pressure_parts.push_back(std::move(p));
    }
  }
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    auto p = part_on<PressurePart>(s);
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      s.place(p.modes, lam, lam);
      p.diag.push_back(column_tail(c, lam, lam, s.side()) * (rule.weights[k] / (2.0 * kPi * lam)));
      p.row.push_back({cplx(s.side() * lam), -kI * lam});
    }
    pz.pressure_parts.push_back(std::move(p));
  }
}

// Stokes double layer (stresslet with per-source normals): the symbol splits into two
// source-side matrices a1 / a2 contracted with (f n^T) and a target-side matrix smat with
// the scalar factors sa, sb and the tail offset `off`.
void dlp_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const Mat2c eye{1.0, 0.0, 0.0, 1.0};
  if (c.periodicity == Periodicity::Doubly) {
    const int base = truncation_order(c, pz.eps);
    const double chi0 = 2.0 * kPi * base / c.d;
    const int M = widen(c, base, chi0 * c.eta * chi0 * c.eta);
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<StressletPart>(s);
      const double side = s.side();
      each_fourier(c, M, false, [&](int m, double alpha) {
        const double a = std::abs(alpha);
        const double sg = m > 0 ? 1.0 : -1.0;
        const cplx Q = strip_q(c, s, a, alpha);
        const cplx amp = strip_tail(Q, a * c.eta) / (2.0 * c.d);
        s.place(p.modes, alpha, a);
        p.a1.push_back(Mat2c{2.0 * kI * sg, -side, -side, 0.0} * amp);
        p.a2.push_back(eye * (-side * amp));
        p.sa.push_back(kI * alpha);
        p.sb.push_back(cplx(-side * a));
        p.smat.push_back(Mat2c{side, kI * sg, kI * sg, -side} * (-amp));
        p.off.push_back(side * tail_moment(Q) * c.eta);
      });
      p.has_m0 = true;
      p.m0_coef = 1.0 / (2.0 * c.d * c.eta);
      pz.stresslet_parts.push_back(std::move(p));
    }
  }
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    const bool west = s.lower;
    auto p = part_on<StressletPart>(s);
    const Mat2c m1 = west ? eye * cplx(-1.0) : eye;
    const Mat2c m2 = west ? Mat2c{0.0, -1.0, -1.0, 2.0 * kI} : Mat2c{0.0, 1.0, 1.0, 2.0 * kI};
    const Mat2c cm = west ? Mat2c{-1.0, kI, kI, 1.0} : Mat2c{1.0, kI, kI, -1.0};
    for (std::size_t k = 0; k < rule.size(); ++k) {
      const double lam = rule.nodes[k];
      const RowSums rows = row_sums(c, lam);
      const cplx even = west ? rows.even : std::conj(rows.even);
      const cplx odd = west ? rows.odd : -std::conj(rows.odd);
      const double amp = rule.weights[k] * column_tail_plain(c, lam) / (2.0 * kPi);
      const cplx sa = west ? cplx(-lam) : cplx(lam), sb = kI * lam;
      const cplx gm = tail_moment_columns(lam * c.d, c.m0);
      s.place(p.modes, lam, lam);
      p.a1.push_back((m1 * even + cm * (c.xi * sa * odd)) * amp);
      p.a2.push_back((m2 * even + cm * (c.xi * sb * odd)) * amp);
      p.sa.push_back(sa);
      p.sb.push_back(sb);
      p.smat.push_back(cm * (-amp * even));
      p.off.push_back((west ? gm : -gm) * c.d);
    }
    pz.stresslet_parts.push_back(std::move(p));
  }
}

// ---------------------------------------------------------------- multipole sources (order l)
// Complex coefficients per source; the symbol of the l-th multipole grows like chi^l, so
// the vertical modes extend past the truncation order (and the symbol's peak) until a mode
// falls below 0.1 eps of the largest, and the half-line rule's truncation moves out
// (multipole_upper).
cplx ipow(cplx z, int l) {
  cplx r{1.0, 0.0};
  for (int i = 0; i < l; ++i) r *= z;
  return r;
}
double fact_lt4(int n) { return n <= 1 ? 1.0 : n == 2 ? 2.0 : 6.0; }

// append modes while `entry(m)` is not yet negligible: |m| past both `base` and `peak`
// and |value| <= 0.1 eps max|value| stops (the first m's up to base always go in)
struct Extender {
  int base, peak;
  double cut, biggest = 0.0;
  bool keep(int mabs, double mag) {
    if (mabs > std::max(base, peak) && mag <= cut * biggest) return false;
    biggest = std::max(biggest, mag);
    return true;
  }
};

void multipole_tables(Periodizer& pz, const QuadratureRule& rule) {
  const UnitCell& c = pz.cell;
  const int l = pz.multipole_order;
  const bool screened = pz.pde == Pde::ModHelmholtz;
  const double beta = pz.beta;
  if (c.periodicity == Periodicity::Doubly) {
    const int base = truncation_order(c, pz.eps);
    for (Direction d : kVertical) {
      const Strip s = Strip::of(c, d);
      auto p = part_on<ScalarPart>(s);
      p.take_real = false;
      const bool south = s.lower;
      if (screened) {
        const int peak = static_cast<int>(std::ceil(l * c.d / (2.0 * kPi * c.eta))) + 1;
        Extender ext{base, peak, 0.1 * pz.eps};
        const cplx pre = ipow(south ? kI : -kI, l) * (kPi / c.d);
        auto add = [&](int m) {
          const double alpha = 2.0 * kPi * m / c.d, chi = std::hypot(alpha, beta);
          const double ratio = south ? (alpha >= 0.0 ? beta / (chi + alpha) : (chi - alpha) / beta)
                                     : (alpha >= 0.0 ? (chi + alpha) / beta : beta / (chi - alpha));
          const cplx v = pre * (std::pow(ratio, l) / chi) * strip_tail(strip_q(c, s, chi, alpha), chi * c.eta);
          if (!ext.keep(std::abs(m), std::abs(v))) return false;
          s.place(p.modes, alpha, chi);
          p.diag.push_back(v);
          return true;
        };
        for (int m = -base; m <= base; ++m) add(m);
        const int step = south ? -1 : 1;  // the growing side of the symbol
        for (int m = step * (base + 1);; m += step) {
          require(std::abs(m) < kModeCap, ErrorCode::NotConverged, "multipole mode extension runs away");
          if (!add(m)) break;
        }
      } else {
        const int peak = static_cast<int>(std::ceil((l - 1) * c.d / (2.0 * kPi * c.eta))) + 1;
        Extender ext{base, peak, 0.1 * pz.eps};
        const cplx pre = ipow((south ? -kI : kI) * (2.0 * kPi / c.d), l) / fact_lt4(l - 1);
        auto add = [&](int m) {  // m > 0 only; the phase sign carries the side
          const double alpha = 2.0 * kPi * m / c.d;
          const cplx Q(alpha * c.eta, -alpha * c.xi);
          const cplx v = pre * std::pow(static_cast<double>(m), l - 1) * strip_tail(Q, alpha * c.eta);
          if (!ext.keep(m, std::abs(v))) return false;
          s.place(p.modes, south ? alpha : -alpha, alpha);
          p.diag.push_back(v);
          return true;
        };
        for (int m = 1; m <= base; ++m) add(m);
        for (int m = base + 1;; ++m) {
          require(m < kModeCap, ErrorCode::NotConverged, "multipole mode extension runs away");
          if (!add(m)) break;
        }
      }
      pz.scalar_parts.push_back(std::move(p));
    }
  }
  for (Direction d : kHorizontal) {
    const Strip s = Strip::of(c, d);
    auto p = part_on<ScalarPart>(s);
    p.take_real = false;
    const bool west = s.lower;
    if (screened) {
      const double side = s.side();
      const cplx pre = (west || l % 2 == 0 ? 1.0 : -1.0) / (2.0 * std::pow(beta, l));
      for (std::size_t k = 0; k < rule.size(); ++k) {
        const double lam = rule.nodes[k], chi = std::hypot(lam, beta);
        for (double lt : {lam, -lam}) {
          const double sym = side * lt >= 0.0 ? chi + side * lt : beta * beta / (chi + std::abs(lt));
          s.place(p.modes, lt, chi);
          p.diag.push_back(pre * std::pow(sym, l) * (rule.weights[k] / chi) * column_tail(c, chi, lt, side));
        }
      }
    } else {
      const double pre = (west || l % 2 == 0) ? 1.0 : -1.0;
      for (std::size_t k = 0; k < rule.size(); ++k) {
        const double lam = rule.nodes[k];
        cplx rows{1.0, 0.0};
        if (c.periodicity == Periodicity::Doubly)
          rows += std::exp(cplx(lam * c.xi, lam * c.eta)) + std::exp(cplx(-lam * c.xi, -lam * c.eta));
        s.place(p.modes, west ? -lam : lam, lam);
        p.diag.push_back(pre * std::pow(lam, l - 1) / fact_lt4(l - 1) * rule.weights[k] * rows *
                         column_tail_plain(c, lam));
      }
    }
    pz.scalar_parts.push_back(std::move(p));
  }
}

// The half-line truncation for a multipole symbol: move lambda_max out (in steps of half an
// oscillation period) until the log-magnitude of the horizontal coefficient is a full
// 0.1 eps below its peak (periodize_multipole.cpp:174-203).
double multipole_upper(Pde pde, double beta, int l, const UnitCell& c, double eps) {
  const double gap = c.m0 * c.d - std::abs(c.xi);
  const double lam0 = 2.0 * kPi / (c.periodicity == Periodicity::Doubly ? 2.0 * c.eta : c.eta);
  auto logmag = [&](double lam) {
    if (pde == Pde::ModHelmholtz) {
      const double chi = std::hypot(lam, beta);
      return l * std::log((chi + lam) / beta) - chi * gap - std::log(chi) - std::log(-std::expm1(-chi * c.d));
    }
    return (l - 1) * std::log(lam) - lam * gap - std::log(-std::expm1(-lam * c.d));
  };
  const QuadratureRule plain = sommerfeld_rule(pde, beta, c, eps);
  const double start = plain.upper > 0.0 ? plain.upper : std::log(1.0 / eps) / c.d;
  // peak over a log-spaced scan of [lam0 / 100, max(start, 4 lam0)]
  const double lo = 1e-2 * lam0, hi = std::max(start, 4.0 * lam0);
  double peak = -1e300;
  for (int i = 0; i < 400; ++i) peak = std::max(peak, logmag(lo * std::pow(hi / lo, i / 399.0)));
  const double floor = peak + std::log(0.1 * eps);
  double up = std::max(start, lam0);
  for (int steps = 0; logmag(up) > floor; ++steps) {
    require(steps < 2000000, ErrorCode::NotConverged, "multipole truncation scan runs away");
    up += 0.5 * lam0;
  }
  return up;
}

}  // namespace

// Theorem 3.1: the smallest M with the vertical tail below eps,
// ceil(d / (2 pi eta) ln(1 / ((1 - e^{-2 pi eta / d}) eps))).
int truncation_order(const UnitCell& cell, double eps) {
  require_eps(eps);
  const double x = 2.0 * kPi * cell.eta / cell.d;
  return static_cast<int>(std::ceil(cell.d / (2.0 * kPi * cell.eta) * std::log(1.0 / (-std::expm1(-x) * eps))));
}

// The bound the theorem gives for order M: e^{-t} / (2 pi (M + 1) (1 - e^{-t}) (1 - e^{-t1})),
// t = 2 pi (M + 1) eta / d, t1 = 2 pi eta / d.
double vertical_tail_bound(const UnitCell& cell, int M) {
  require(M >= 1, ErrorCode::InvalidOrder, "the tail bound needs M >= 1");
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

// periodize.hpp:119 (reference make_periodizer): every strip of the kernel's symbol; the
// Stokes family adds its pressure tables, and reuses the unscreened rule for both symbols.
Periodizer make_periodizer(Pde pde, double beta, const UnitCell& cell, double eps) {
  require_eps(eps);
  const bool screened = pde == Pde::ModHelmholtz || pde == Pde::ModStokes;
  if (screened) require(beta > 0.0, ErrorCode::MissingBeta, "a screened kernel needs beta > 0");
  Periodizer pz;
  pz.pde = pde;
  pz.beta = screened ? beta : 0.0;
  pz.cell = cell;
  pz.eps = eps;
  pz.requires_neutrality = screened ? beta < kUnscreenedBeta : true;
  switch (pde) {
    case Pde::Poisson:
    case Pde::ModHelmholtz:
      scalar_tables(pz, certified_rule(pde, pz.beta, cell, eps));
      break;
    case Pde::Stokes:
    case Pde::ModStokes: {
      const QuadratureRule rule = certified_rule(Pde::Stokes, 0.0, cell, eps);
      if (pde == Pde::Stokes)
        stokes_tables(pz, rule);
      else
        mod_stokes_tables(pz, rule);
      pressure_tables(pz, rule);
      break;
    }
  }
  return pz;
}

// periodize.hpp:122 (reference make_stokes_dlp_periodizer)
Periodizer make_stokes_dlp_periodizer(const UnitCell& cell, double eps) {
  require_eps(eps);
  Periodizer pz;
  pz.pde = Pde::Stokes;
  pz.cell = cell;
  pz.eps = eps;
  pz.dlp = true;
  pz.requires_neutrality = true;
  dlp_tables(pz, certified_rule(Pde::Stokes, 0.0, cell, eps));
  return pz;
}

// periodize.hpp:127 (reference make_multipole_periodizer): orders 1..4 of the scalar kernels
Periodizer make_multipole_periodizer(Pde pde, double beta, int l, const UnitCell& cell, double eps) {
  require_eps(eps);
  require(pde == Pde::Poisson || pde == Pde::ModHelmholtz, ErrorCode::Unsupported,
          "multipole sources exist for the scalar kernels only");
  require(l >= 1 && l <= 4, ErrorCode::OrderOutOfRange, "multipole order must lie in 1..4");
  const bool screened = pde == Pde::ModHelmholtz;
  if (screened) require(beta > 0.0, ErrorCode::MissingBeta, "a screened kernel needs beta > 0");
  Periodizer pz;
  pz.pde = pde;
  pz.beta = screened ? beta : 0.0;
  pz.cell = cell;
  pz.eps = eps;
  pz.multipole_order = l;
  pz.requires_neutrality = pde == Pde::Poisson && l == 1;
  const double up = multipole_upper(pde, pz.beta, l, cell, eps);
  multipole_tables(pz, certified_rule(pde, pz.beta, cell, eps, up));
  return pz;
}

}  // namespace periwave
