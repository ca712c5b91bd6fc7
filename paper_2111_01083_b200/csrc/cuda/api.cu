// The drop-in C++ API (include/periwave/periwave.hpp) over the C-ABI engine:
// apply_far / total_field / FreeSpaceEvaluator::accumulate / choose_path /
// NUFFT / brute_force_far / periodicity_residual with the reference's
// signatures and error behaviour (periwave::Error thrown with the same codes).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "periwave/periwave.hpp"
#include "periwave_b200.h"

struct pwb_periodizer;
namespace pwb {
pwb_periodizer* wrap_periodizer(const periwave::Periodizer& pz);
}

namespace periwave {
namespace {

[[noreturn]] void rethrow(int code) {
  const std::string msg = pwb_last_error();
  if (code >= 1 && code <= 19) throw Error(static_cast<ErrorCode>(code - 1), msg);
  throw std::runtime_error("periwave-b200: " + msg);
}

void check(int code) {
  if (code != PWB_OK) rethrow(code);
}

enum class K { Scalar, Velocity, Multipole };
K kind(const Periodizer& pz) {
  if (pz.multipole_order >= 1) return K::Multipole;
  if (pz.pde == Pde::Stokes || pz.pde == Pde::ModStokes) return K::Velocity;
  return K::Scalar;
}

// ---- one device plan per distinct periodizer
// The reference passes the periodizer by const& to every call (apply.hpp:58-60); building a
// device plan (stream, mode tables, NUFFT setup, workspaces) per call would cost more than a
// small evaluation and all of a repeated one. The cache keys a wrapped periodizer by its
// full content (every table byte), so equal periodizers share one plan and a modified copy
// gets its own. A handful of recent entries are kept (LRU); the cache is intentionally never
// destroyed (its plans hold CUDA resources that must not be freed during static teardown).
class Bytes {
 public:
  template <class T>
  void pod(const T& v) {
    static_assert(std::is_trivially_copyable_v<T>);
    const auto* p = reinterpret_cast<const unsigned char*>(&v);
    b_.insert(b_.end(), p, p + sizeof(T));
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    pod(v.size());
    if (!v.empty()) {
      const auto* p = reinterpret_cast<const unsigned char*>(v.data());
      b_.insert(b_.end(), p, p + v.size() * sizeof(T));
    }
  }
  void modes(const ModeSet& m) {
    pod(m.axis);
    vec(m.phase);
    vec(m.decay_t);
    vec(m.decay_s);
    vec(m.shift_t);
    vec(m.shift_s);
  }
  std::vector<unsigned char> take() { return std::move(b_); }

 private:
  std::vector<unsigned char> b_;
};

std::vector<unsigned char> content_key(const Periodizer& pz) {
  Bytes k;
  k.pod(pz.pde);
  k.pod(pz.beta);
  k.pod(pz.cell.d);
  k.pod(pz.cell.xi);
  k.pod(pz.cell.eta);
  k.pod(pz.cell.periodicity);
  k.pod(pz.cell.m0);
  k.pod(pz.eps);
  k.pod(pz.dlp);
  k.pod(pz.multipole_order);
  k.pod(pz.requires_neutrality);
  k.pod(pz.scalar_parts.size());
  for (const auto& p : pz.scalar_parts) {
    k.pod(p.dir);
    k.modes(p.modes);
    k.vec(p.diag);
    k.pod(p.take_real);
    k.pod(p.has_m0);
    k.pod(p.m0_coef);
  }
  k.pod(pz.block_parts.size());
  for (const auto& p : pz.block_parts) {
    k.pod(p.dir);
    k.modes(p.modes);
    k.vec(p.diag_a);
    k.vec(p.diag_b);
    k.pod(p.three_term);
    k.pod(p.take_real);
    k.pod(p.has_m0);
    k.pod(p.m0_mat);
  }
  k.pod(pz.pressure_parts.size());
  for (const auto& p : pz.pressure_parts) {
    k.pod(p.dir);
    k.modes(p.modes);
    k.vec(p.diag);
    k.vec(p.row);
    k.pod(p.has_m0);
    k.pod(p.m0_coef);
    k.pod(p.m0_row);
  }
  k.pod(pz.stresslet_parts.size());
  for (const auto& p : pz.stresslet_parts) {
    k.pod(p.dir);
    k.modes(p.modes);
    k.vec(p.a1);
    k.vec(p.a2);
    k.vec(p.smat);
    k.vec(p.sa);
    k.vec(p.sb);
    k.vec(p.off);
    k.pod(p.has_m0);
    k.pod(p.m0_coef);
  }
  return k.take();
}

class PlanCache {
 public:
  static PlanCache& instance() {
    static PlanCache* c = new PlanCache;  // never destroyed (see above)
    return *c;
  }
  std::shared_ptr<pwb_periodizer> get(const Periodizer& pz) {
    std::vector<unsigned char> key = content_key(pz);
    std::lock_guard<std::mutex> g(mu_);
    ++tick_;
    for (auto& e : entries_)
      if (e.key == key) {
        e.last = tick_;
        return e.h;
      }
    if (entries_.size() >= capacity()) {
      auto lru = std::min_element(entries_.begin(), entries_.end(),
                                  [](const Entry& a, const Entry& b) { return a.last < b.last; });
      entries_.erase(lru);  // freed when the last call using it returns
    }
    entries_.push_back(Entry{std::move(key), std::shared_ptr<pwb_periodizer>(pwb::wrap_periodizer(pz),
                                                                             pwb_periodizer_free),
                             tick_});
    return entries_.back().h;
  }
 private:
  struct Entry {
    std::vector<unsigned char> key;
    std::shared_ptr<pwb_periodizer> h;
    unsigned long long last;
  };
  static size_t capacity() {
    const char* e = std::getenv("PWB_PLAN_CACHE");
    const long v = e ? std::strtol(e, nullptr, 10) : 8;
    return static_cast<size_t>(std::max(1L, v));
  }
  std::mutex mu_;
  std::vector<Entry> entries_;
  unsigned long long tick_ = 0;
};

// The cached handle of `pz` (shared between calls with equal periodizers).
struct Handle {
  std::shared_ptr<pwb_periodizer> keep;
  pwb_periodizer* h;
  explicit Handle(const Periodizer& pz) : keep(PlanCache::instance().get(pz)), h(keep.get()) {}
};

pwb_system system_of(const ParticleSystem& s) {
  pwb_system o{};
  o.n_src = s.sources.size();
  o.n_tgt = s.targets.size();
  o.sources = reinterpret_cast<const double*>(s.sources.data());
  o.charges = s.charges.empty() ? nullptr : s.charges.data();
  o.forces = s.forces.empty() ? nullptr : reinterpret_cast<const double*>(s.forces.data());
  o.normals = s.normals.empty() ? nullptr : reinterpret_cast<const double*>(s.normals.data());
  o.coefficients = s.coefficients.empty() ? nullptr : reinterpret_cast<const double*>(s.coefficients.data());
  o.targets = reinterpret_cast<const double*>(s.targets.data());
  o.memory = PWB_MEM_HOST;
  return o;
}

pwb_options options_of(const ApplyOptions& a) {
  pwb_options o;
  pwb_options_default(&o);
  o.path = static_cast<int>(a.path);
  o.threads = a.threads;
  o.with_pressure = a.with_pressure ? 1 : 0;
  o.nufft_eps = a.nufft_eps;
  o.with_gradient = a.with_gradient ? 1 : 0;
  o.device = a.device;
  o.stream = a.stream;
  return o;
}

bool lengths_ok(const ParticleSystem& s) {
  const size_t ns = s.sources.size();
  auto ok = [ns](size_t n) { return n == 0 || n == ns; };
  return ok(s.charges.size()) && ok(s.forces.size()) && ok(s.normals.size()) && ok(s.coefficients.size());
}

// validate_system (cell.cpp:77-94) for a call that goes on to the device: the C-ABI call
// checks cell membership and unit normals on the device (same rules and error codes,
// engine.cu Plan::validate), so the O(N) host scan -- ~30 ms at N = 1e6, 5 % of a c4 step --
// is not repeated on the success path. A strength vector of the wrong length, which the
// pointer interface cannot see, is checked here first; and when the device call fails, the
// host scan runs before the error is rethrown, so the error raised is the one the reference
// raises (its validate_system comes before every other check, apply.cpp:417-430).
template <class F>
void validated_device_call(const UnitCell& cell, const ParticleSystem& s, F&& call) {
  if (!lengths_ok(s)) validate_system(cell, s);
  try {
    call();
  } catch (...) {
    validate_system(cell, s);
    throw;
  }
}

void check_lengths(const ParticleSystem& s) {
  const size_t ns = s.sources.size();
  auto ok = [ns](size_t n) { return n == 0 || n == ns; };
  require(ok(s.charges.size()), ErrorCode::LengthMismatch, "charges length does not match sources");
  require(ok(s.forces.size()), ErrorCode::LengthMismatch, "forces length does not match sources");
  require(ok(s.normals.size()), ErrorCode::LengthMismatch, "normals length does not match sources");
  require(ok(s.coefficients.size()), ErrorCode::LengthMismatch, "coefficients length does not match sources");
}

// sizes FieldResult like apply.cpp:395-405, optionally keeping existing values
pwb_field field_of(const Periodizer& pz, const ApplyOptions& opt, size_t nt, FieldResult& f, bool keep) {
  auto fit = [&](auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    if (!keep || v.size() != nt) v.assign(nt, T{});
  };
  pwb_field o{};
  o.memory = PWB_MEM_HOST;
  switch (kind(pz)) {
    case K::Multipole:
      fit(f.complex_scalar);
      o.complex_scalar = reinterpret_cast<double*>(f.complex_scalar.data());
      break;
    case K::Velocity:
      fit(f.velocity);
      o.velocity = reinterpret_cast<double*>(f.velocity.data());
      if (opt.with_pressure) {
        fit(f.pressure);
        o.pressure = f.pressure.data();
      }
      break;
    case K::Scalar:
      fit(f.scalar);
      o.scalar = f.scalar.data();
      if (opt.with_gradient) {
        fit(f.gradient);
        o.gradient = reinterpret_cast<double*>(f.gradient.data());
      }
      break;
  }
  return o;
}

}  // namespace

ApplyPath choose_path(const Periodizer& pz, std::size_t n_src, std::size_t n_tgt) {  // apply.cpp:409-415
  const bool scalar_kind = (pz.pde == Pde::Poisson || pz.pde == Pde::ModHelmholtz) && pz.multipole_order == 0 && !pz.dlp;
  if (scalar_kind && pz.rank() > 256 && n_src + n_tgt > 4096 && fast_nufft_available()) return ApplyPath::Accelerated;
  return ApplyPath::Direct;
}

FieldResult apply_far(const Periodizer& pz, const ParticleSystem& sys, const ApplyOptions& opt) {
  Handle h(pz);
  pwb_system s = system_of(sys);
  pwb_options o = options_of(opt);
  FieldResult out;
  pwb_field f = field_of(pz, opt, sys.targets.size(), out, false);
  validated_device_call(pz.cell, sys, [&] { check(pwb_apply_far(h.h, &s, &o, &f)); });
  out.accelerated = f.accelerated != 0;
  return out;
}

void FreeSpaceEvaluator::accumulate(const Periodizer& pz, const ParticleSystem& sys, Vec2 shift, bool identity_shift,
                                    const ApplyOptions& opt, FieldResult& out) const {
  check_lengths(sys);
  Handle h(pz);
  pwb_system s = system_of(sys);
  pwb_options o = options_of(opt);
  pwb_field f = field_of(pz, opt, sys.targets.size(), out, true);
  check(pwb_accumulate(h.h, &s, shift.x, shift.y, identity_shift ? 1 : 0, &o, &f));
}

FieldResult total_field(const Periodizer& pz, const ParticleSystem& sys, const ApplyOptions& opt,
                        const FreeSpaceEvaluator* near_eval) {
  if (near_eval) {  // user plug-in: honour it image by image (apply.cpp:548-556)
    FieldResult out = apply_far(pz, sys, opt);
    for (const LatticeTranslation& tr : near_translations(pz.cell))
      near_eval->accumulate(pz, sys, tr.shift, tr.m == 0 && tr.n == 0, opt, out);
    return out;
  }
  Handle h(pz);
  pwb_system s = system_of(sys);
  pwb_options o = options_of(opt);
  FieldResult out;
  pwb_field f = field_of(pz, opt, sys.targets.size(), out, false);
  validated_device_call(pz.cell, sys, [&] { check(pwb_total_field(h.h, &s, &o, &f)); });
  out.accelerated = f.accelerated != 0;
  return out;
}

bool fast_nufft_available() { return pwb_fast_nufft_available() != 0; }

void nufft_type1(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& c,
                 std::size_t nmodes, std::vector<cplx>& f) {
  require(x.size() == c.size(), ErrorCode::LengthMismatch, "points and strengths must have equal length");
  f.assign(nmodes, cplx{0.0, 0.0});
  check(pwb_nufft_type1(static_cast<int>(backend), eps, x.size(), x.data(), reinterpret_cast<const double*>(c.data()),
                        nmodes, reinterpret_cast<double*>(f.data()), PWB_MEM_HOST, nullptr));
}

void nufft_type2(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& f,
                 std::vector<cplx>& c) {
  c.assign(x.size(), cplx{0.0, 0.0});
  check(pwb_nufft_type2(static_cast<int>(backend), eps, x.size(), x.data(), f.size(),
                        reinterpret_cast<const double*>(f.data()), reinterpret_cast<double*>(c.data()), PWB_MEM_HOST,
                        nullptr));
}

void nufft_type3(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& c,
                 const std::vector<double>& s, std::vector<cplx>& f) {
  require(x.size() == c.size(), ErrorCode::LengthMismatch, "points and strengths must have equal length");
  f.assign(s.size(), cplx{0.0, 0.0});
  check(pwb_nufft_type3(static_cast<int>(backend), eps, x.size(), x.data(), reinterpret_cast<const double*>(c.data()),
                        s.size(), s.data(), reinterpret_cast<double*>(f.data()), PWB_MEM_HOST, nullptr));
}

// ---------------------------------------------------------------- validation tools (oracle.cpp)
namespace {

bool near_image(const UnitCell& c, int m, int n) {
  if (c.periodicity == Periodicity::Doubly) return std::abs(m) <= c.m0 && std::abs(n) <= 1;
  return n == 0 && std::abs(m) <= 1;
}

// half of shell max(|m|,|n|) == s, the other half being its negation (oracle.cpp:20-33)
std::vector<std::pair<int, int>> shell_half(const UnitCell& c, int s) {
  std::vector<std::pair<int, int>> h;
  if (c.periodicity == Periodicity::Singly) {
    if (!near_image(c, s, 0)) h.emplace_back(s, 0);
    return h;
  }
  for (int m = -s; m <= s; ++m)
    if (!near_image(c, m, s)) h.emplace_back(m, s);
  for (int n = 1; n < s; ++n)
    if (!near_image(c, s, n)) h.emplace_back(s, n);
  for (int n = 0; n < s; ++n)
    if (!near_image(c, s, -n)) h.emplace_back(s, -n);
  return h;
}

double abs_max(const FieldResult& f) {
  double m = 0.0;
  for (double v : f.scalar) m = std::max(m, std::abs(v));
  for (const Vec2& v : f.velocity) m = std::max({m, std::abs(v.x), std::abs(v.y)});
  for (double v : f.pressure) m = std::max(m, std::abs(v));
  for (const cplx& v : f.complex_scalar) m = std::max(m, std::abs(v));
  return m;
}

double diff_max(const FieldResult& a, const FieldResult& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.scalar.size(); ++i) m = std::max(m, std::abs(a.scalar[i] - b.scalar[i]));
  for (size_t i = 0; i < a.velocity.size(); ++i)
    m = std::max({m, std::abs(a.velocity[i].x - b.velocity[i].x), std::abs(a.velocity[i].y - b.velocity[i].y)});
  for (size_t i = 0; i < a.pressure.size(); ++i) m = std::max(m, std::abs(a.pressure[i] - b.pressure[i]));
  for (size_t i = 0; i < a.complex_scalar.size(); ++i)
    m = std::max(m, std::abs(a.complex_scalar[i] - b.complex_scalar[i]));
  return m;
}

void components(const FieldResult& f, size_t l, std::vector<double>& out) {
  out.clear();
  if (!f.scalar.empty()) out.push_back(f.scalar[l]);
  if (!f.velocity.empty()) {
    out.push_back(f.velocity[l].x);
    out.push_back(f.velocity[l].y);
  }
  if (!f.pressure.empty()) out.push_back(f.pressure[l]);
  if (!f.complex_scalar.empty()) {
    out.push_back(f.complex_scalar[l].real());
    out.push_back(f.complex_scalar[l].imag());
  }
}

}  // namespace

// oracle.cpp:83-110: shell-by-shell +- paired lattice sum, early stop after
// three quiet shells at 1e-18.
FieldResult brute_force_far(const Periodizer& pz, const ParticleSystem& sys, int shells, const ApplyOptions& opt) {
  validate_system(pz.cell, sys);
  FreeSpaceEvaluator eval;
  FieldResult out, before;
  int quiet = 0;
  for (int s = 1; s <= shells; ++s) {
    const auto half = shell_half(pz.cell, s);
    if (half.empty()) continue;
    before = out;
    for (auto [m, n] : half) {
      const Vec2 plus = pz.cell.e1() * double(m) + pz.cell.e2() * double(n);
      eval.accumulate(pz, sys, plus, false, opt, out);
      eval.accumulate(pz, sys, Vec2{-plus.x, -plus.y}, false, opt, out);
    }
    if (before.scalar.empty() && before.velocity.empty() && before.pressure.empty() && before.complex_scalar.empty())
      continue;
    const double scale = std::max(abs_max(out), 1e-300);
    if (diff_max(out, before) <= 1e-18 * scale) {
      if (++quiet >= 3) break;
    } else {
      quiet = 0;
    }
  }
  return out;
}

// oracle.cpp:112-173: face jumps vs the mean-removed RMS.
ResidualReport periodicity_residual(const Periodizer& pz, const ParticleSystem& sys, int samples_per_side,
                                    const ApplyOptions& opt) {
  require(samples_per_side >= 1, ErrorCode::NonPositiveDimension,
          "periodicity_residual requires at least one sample per side");
  const UnitCell& c = pz.cell;
  const size_t sps = static_cast<size_t>(samples_per_side);
  const bool doubly = c.periodicity == Periodicity::Doubly;
  ParticleSystem probe = sys;
  probe.targets.clear();
  const Vec2 e1 = c.e1(), e2 = c.e2();
  for (size_t v = 0; v < sps; ++v) {
    const double t = (double(v) + 0.5) / double(sps) - 0.5;
    probe.targets.push_back(e2 * t - e1 * 0.5);
    probe.targets.push_back(e2 * t + e1 * 0.5);
  }
  if (doubly)
    for (size_t v = 0; v < sps; ++v) {
      const double t = (double(v) + 0.5) / double(sps) - 0.5;
      probe.targets.push_back(e1 * t - e2 * 0.5);
      probe.targets.push_back(e1 * t + e2 * 0.5);
    }
  const FieldResult f = total_field(pz, probe, opt);
  std::vector<double> comp;
  components(f, 0, comp);
  const size_t nc = comp.size(), np = probe.targets.size();
  std::vector<double> vals(np * nc);
  for (size_t l = 0; l < np; ++l) {
    components(f, l, comp);
    for (size_t i = 0; i < nc; ++i) vals[l * nc + i] = comp[i];
  }
  auto rms_jump = [&](size_t base) {
    double acc = 0.0;
    for (size_t v = 0; v < sps; ++v)
      for (size_t i = 0; i < nc; ++i) {
        const double d = vals[(base + 2 * v + 1) * nc + i] - vals[(base + 2 * v) * nc + i];
        acc += d * d;
      }
    return std::sqrt(acc / double(sps * nc));
  };
  ResidualReport rep;
  rep.e1 = rms_jump(0);
  if (doubly) rep.e2 = rms_jump(2 * sps);
  double acc = 0.0;
  for (size_t i = 0; i < nc; ++i) {
    double mean = 0.0;
    for (size_t l = 0; l < np; ++l) mean += vals[l * nc + i];
    mean /= double(np);
    for (size_t l = 0; l < np; ++l) {
      const double d = vals[l * nc + i] - mean;
      acc += d * d;
    }
  }
  rep.scale = std::sqrt(acc / double(np * nc));
  return rep;
}

}  // namespace periwave
