// periwave-b200: command-line front end over the drop-in C++ API.
//
// Mirrors the reference tool's `apply` and `validate` subcommands
// (/root/reference/proj/tools/periwave_cli.cpp:328-361 and :255-326): the same
// options, the same text record formats ('x y q' / 'x y fx fy [nx ny]' sources,
// 'x y' targets, '#' comments, blank lines skipped), the same %.17g field lines
// and the same exit codes (0 ok, 1 validate gate failed, 2 error with an
// "error: <path>:<line>: ..." diagnostic). Every N-scaling step runs through
// libperiwave_b200.so on the GPU; this file only parses, wraps and prints.
// The reference's `bench` subcommand is replaced by bench.py.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "periwave/periwave.hpp"

namespace {

using namespace periwave;
using Clock = std::chrono::steady_clock;

struct Args {
  std::string cmd;
  std::string pde = "poisson";
  double beta = 0.0;
  std::vector<double> cell;            // d, xi, eta
  std::vector<double> aspects{1.0};
  bool aspects_given = false, theta_given = false;
  double theta = 90.0;
  int periodicity = 2;
  double eps = 1e-12;
  int n_src = 4000;
  std::uint64_t seed = 1234;
  std::string accel = "auto";
  int samples = 500;
  std::string out;
  int threads = 1;
  bool pressure = false;
  std::string dump_sources, dump_fields;
  std::vector<std::string> positional;
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

double to_double(const std::string& flag, const std::string& s) {
  char* end = nullptr;
  double v = std::strtod(s.c_str(), &end);
  if (s.empty() || *end != '\0') throw UsageError(flag + ": not a number: " + s);
  return v;
}

long long to_int(const std::string& flag, const std::string& s) {
  char* end = nullptr;
  long long v = std::strtoll(s.c_str(), &end, 10);
  if (s.empty() || *end != '\0') throw UsageError(flag + ": not an integer: " + s);
  return v;
}

std::vector<double> to_list(const std::string& flag, const std::string& s) {
  std::vector<double> v;
  std::size_t p = 0;
  while (p <= s.size()) {
    std::size_t q = s.find(',', p);
    if (q == std::string::npos) q = s.size();
    v.push_back(to_double(flag, s.substr(p, q - p)));
    p = q + 1;
  }
  return v;
}

Args parse_args(int argc, char** argv) {
  Args a;
  if (argc < 2) throw UsageError("expected a subcommand: apply | validate");
  a.cmd = argv[1];
  if (a.cmd != "apply" && a.cmd != "validate") throw UsageError("unknown subcommand: " + a.cmd);
  for (int i = 2; i < argc; ++i) {
    std::string f = argv[i];
    if (f.rfind("--", 0) != 0) {
      a.positional.push_back(f);
      continue;
    }
    std::string val;
    std::size_t eq = f.find('=');
    if (eq != std::string::npos) {
      val = f.substr(eq + 1);
      f = f.substr(0, eq);
    }
    if (f == "--pressure") {
      a.pressure = true;
      continue;
    }
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw UsageError(f + ": missing value");
      val = argv[++i];
    }
    if (f == "--pde") {
      if (val != "poisson" && val != "mhelm" && val != "stokes" && val != "mstokes")
        throw UsageError("--pde: one of poisson, mhelm, stokes, mstokes");
      a.pde = val;
    } else if (f == "--beta") {
      a.beta = to_double(f, val);
    } else if (f == "--cell") {
      a.cell = to_list(f, val);
      if (a.cell.size() != 3) throw UsageError("--cell: expected d,xi,eta");
    } else if (f == "--aspect") {
      a.aspects = to_list(f, val);
      a.aspects_given = true;
    } else if (f == "--theta") {
      a.theta = to_double(f, val);
      a.theta_given = true;
    } else if (f == "--periodicity") {
      a.periodicity = static_cast<int>(to_int(f, val));
      if (a.periodicity != 1 && a.periodicity != 2) throw UsageError("--periodicity: 1 or 2");
    } else if (f == "--eps") {
      a.eps = to_double(f, val);
    } else if (f == "--n-src") {
      a.n_src = static_cast<int>(to_int(f, val));
      if (a.n_src <= 0) throw UsageError("--n-src: must be positive");
    } else if (f == "--seed") {
      a.seed = static_cast<std::uint64_t>(to_int(f, val));
    } else if (f == "--accel") {
      if (val != "auto" && val != "direct" && val != "nufft") throw UsageError("--accel: auto, direct or nufft");
      a.accel = val;
    } else if (f == "--samples") {
      a.samples = static_cast<int>(to_int(f, val));
      if (a.samples <= 0) throw UsageError("--samples: must be positive");
    } else if (f == "--out") {
      a.out = val;
    } else if (f == "--threads") {
      a.threads = static_cast<int>(to_int(f, val));
    } else if (f == "--dump-sources" && a.cmd == "validate") {
      a.dump_sources = val;
    } else if (f == "--dump-fields" && a.cmd == "validate") {
      a.dump_fields = val;
    } else {
      throw UsageError("unknown option for " + a.cmd + ": " + f);
    }
  }
  if (!a.cell.empty() && (a.aspects_given || a.theta_given))
    throw UsageError("--cell excludes --aspect and --theta");
  if (a.cmd == "apply" && a.positional.size() != 2) throw UsageError("apply: expected <sources> <targets>");
  if (a.cmd == "validate" && !a.positional.empty()) throw UsageError("validate takes no positional arguments");
  return a;
}

Pde pde_of(const std::string& s) {
  if (s == "poisson") return Pde::Poisson;
  if (s == "mhelm") return Pde::ModHelmholtz;
  if (s == "stokes") return Pde::Stokes;
  return Pde::ModStokes;
}

bool is_scalar(Pde p) { return p == Pde::Poisson || p == Pde::ModHelmholtz; }

ApplyOptions options_of(const Args& a, bool with_pressure) {
  ApplyOptions o;
  o.path = a.accel == "direct" ? ApplyPath::Direct : a.accel == "nufft" ? ApplyPath::Accelerated : ApplyPath::Auto;
  o.threads = a.threads;
  o.with_pressure = with_pressure;
  return o;
}

// Explicit --cell, else the aspect/theta family of the reference tool (cli.cpp:78-92).
UnitCell cell_of(const Args& a, double A) {
  const Periodicity per = a.periodicity == 1 ? Periodicity::Singly : Periodicity::Doubly;
  if (a.cell.size() == 3) return make_unit_cell(a.cell[0], a.cell[1], a.cell[2], per);
  require(A >= 1.0, ErrorCode::NonPositiveDimension, "aspect must be >= 1");
  const bool right = std::abs(a.theta - 90.0) < 1e-9;
  if (per == Periodicity::Singly) {
    require(right, ErrorCode::Unsupported, "skew strips need an explicit --cell d,xi,eta");
    return make_unit_cell(1.0, 0.0, A, per);
  }
  const double eta = 1.0 / A, th = a.theta * kPi / 180.0;
  return make_unit_cell(1.0, right ? 0.0 : eta * std::cos(th) / std::sin(th), eta, per);
}

// Integer lattice steps along the periodic directions; inside points stay bit-identical.
Vec2 wrap(const UnitCell& cell, Vec2 p) {
  const Vec2 c = cell_coords(cell, p);
  const double k1 = std::nearbyint(c.x);
  const double k2 = cell.periodicity == Periodicity::Doubly ? std::nearbyint(c.y) : 0.0;
  if (k1 == 0.0 && k2 == 0.0) return p;
  return p - cell.e1() * k1 - cell.e2() * k2;
}

// ------------------------------------------------------------------ text records
std::vector<std::vector<double>> read_records(const std::string& path) {
  std::ifstream in(path);
  require(in.good(), ErrorCode::ParseError, path + ": cannot open");
  std::vector<std::vector<double>> rows;
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    std::istringstream s(line.substr(0, line.find('#')));
    std::vector<double> v;
    double x;
    while (s >> x) v.push_back(x);
    if (!s.eof()) fail(ErrorCode::ParseError, path + ":" + std::to_string(no) + ": malformed number");
    if (v.empty()) continue;
    v.push_back(static_cast<double>(no));  // line number rides along for diagnostics
    rows.push_back(std::move(v));
  }
  return rows;
}

struct Sources {
  std::vector<Vec2> x, f, n;
  std::vector<double> q;
  int cols = 0;
};

Sources read_sources(const std::string& path) {
  Sources s;
  for (const auto& r : read_records(path)) {
    const int cols = static_cast<int>(r.size()) - 1;
    const std::string at = path + ":" + std::to_string(static_cast<long long>(r.back()));
    if (cols != 3 && cols != 4 && cols != 6)
      fail(ErrorCode::ParseError, at + ": expected 'x y q', 'x y fx fy' or 'x y fx fy nx ny'");
    if (s.cols == 0) s.cols = cols;
    if (cols != s.cols) fail(ErrorCode::ParseError, at + ": inconsistent column count");
    s.x.push_back({r[0], r[1]});
    if (cols == 3) s.q.push_back(r[2]);
    if (cols >= 4) s.f.push_back({r[2], r[3]});
    if (cols == 6) s.n.push_back({r[4], r[5]});
  }
  return s;
}

std::vector<Vec2> read_targets(const std::string& path) {
  std::vector<Vec2> t;
  for (const auto& r : read_records(path)) {
    if (r.size() != 3)
      fail(ErrorCode::ParseError, path + ":" + std::to_string(static_cast<long long>(r.back())) + ": expected 'x y'");
    t.push_back({r[0], r[1]});
  }
  return t;
}

std::FILE* open_out(const std::string& path) {
  if (path.empty()) return stdout;
  std::FILE* f = std::fopen(path.c_str(), "w");
  require(f != nullptr, ErrorCode::ParseError, path + ": cannot open for writing");
  return f;
}

void print_fields(std::FILE* out, const std::vector<Vec2>& at, const FieldResult& r, bool with_pressure) {
  for (std::size_t l = 0; l < at.size(); ++l) {
    if (!r.scalar.empty()) {
      std::fprintf(out, "%.17g %.17g %.17g\n", at[l].x, at[l].y, r.scalar[l]);
      continue;
    }
    std::fprintf(out, "%.17g %.17g %.17g %.17g", at[l].x, at[l].y, r.velocity[l].x, r.velocity[l].y);
    if (with_pressure) std::fprintf(out, " %.17g", r.pressure[l]);
    std::fputc('\n', out);
  }
}

// ------------------------------------------------------------------ apply
int run_apply(const Args& a) {
  const UnitCell cell = cell_of(a, a.aspects.empty() ? 1.0 : a.aspects[0]);
  const Pde pde = pde_of(a.pde);
  const std::string& sp = a.positional[0];
  Sources s = read_sources(sp);
  require(s.cols == 0 || !is_scalar(pde) || s.cols == 3, ErrorCode::ParseError, sp + ": scalar kernels take 'x y q' records");
  require(s.cols == 0 || is_scalar(pde) || s.cols >= 4, ErrorCode::ParseError,
          sp + ": vector kernels take 'x y fx fy [nx ny]' records");
  require(s.cols != 6 || pde == Pde::Stokes, ErrorCode::Unsupported, "stresslet densities are Stokes-only");
  const std::vector<Vec2> targets = read_targets(a.positional[1]);

  ParticleSystem sys;
  for (const Vec2& p : s.x) sys.sources.push_back(wrap(cell, p));
  for (const Vec2& p : targets) sys.targets.push_back(wrap(cell, p));
  sys.charges = std::move(s.q);
  sys.forces = std::move(s.f);
  sys.normals = std::move(s.n);

  const Periodizer pz = s.cols == 6 ? make_stokes_dlp_periodizer(cell, a.eps) : make_periodizer(pde, a.beta, cell, a.eps);
  const ApplyOptions opt = options_of(a, a.pressure && !is_scalar(pde) && s.cols != 6);
  const FieldResult r = total_field(pz, sys, opt);
  std::FILE* out = open_out(a.out);
  print_fields(out, targets, r, opt.with_pressure);  // coordinates echoed as given
  if (out != stdout) std::fclose(out);
  return 0;
}

// ------------------------------------------------------------------ validate
ParticleSystem generated_system(const UnitCell& cell, bool scalar, bool neutral, int n, Rng& rng) {
  ParticleSystem sys;
  sys.sources.reserve(n);
  for (int j = 0; j < n; ++j) {
    const double u = rng.uniform(-0.5, 0.5), v = rng.uniform(-0.5, 0.5);
    sys.sources.push_back(cell.e1() * u + cell.e2() * v);
  }
  if (scalar) {
    double mean = 0.0;
    for (int j = 0; j < n; ++j) {
      sys.charges.push_back(rng.uniform(-1.0, 1.0));
      mean += sys.charges.back() / n;
    }
    if (neutral)
      for (double& q : sys.charges) q -= mean;
  } else {
    Vec2 mean;
    for (int j = 0; j < n; ++j) {
      sys.forces.push_back({rng.uniform(-1.0, 1.0), rng.uniform(-1.0, 1.0)});
      mean += sys.forces.back() * (1.0 / n);
    }
    if (neutral)
      for (Vec2& f : sys.forces) f = f - mean;
  }
  return sys;
}

double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

std::string jnum(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string jstr(const std::string& s) { return "\"" + s + "\""; }

int run_validate(const Args& a) {
  const bool fixed = a.cell.size() == 3;
  const std::vector<double> sweep = fixed ? std::vector<double>{0.0} : a.aspects;
  std::vector<std::string> rows, failures;
  std::printf("%8s %8s %7s %9s %9s %9s %9s %9s %11s\n", "A", "rank", "path", "t_build", "t_per", "t_near", "t_total",
              "t_free", "Error");
  for (double A : sweep) {
    const UnitCell cell = cell_of(a, A);
    Clock::time_point t0 = Clock::now();
    const Periodizer pz = make_periodizer(pde_of(a.pde), a.beta, cell, a.eps);
    const double t_build = seconds_since(t0);
    Rng rng(a.seed);
    ParticleSystem sys = generated_system(cell, is_scalar(pz.pde), pz.requires_neutrality, a.n_src, rng);
    sys.targets = sys.sources;
    const ApplyOptions opt = options_of(a, false);
    const ApplyOptions opt_field = options_of(a, a.pressure && !is_scalar(pz.pde));

    t0 = Clock::now();
    (void)apply_far(pz, sys, opt);
    const double t_per = seconds_since(t0);
    t0 = Clock::now();
    const FieldResult total = total_field(pz, sys, opt_field);
    const double t_total = seconds_since(t0);
    const double t_near = std::max(0.0, t_total - t_per);
    FieldResult free_field;
    t0 = Clock::now();
    FreeSpaceEvaluator().accumulate(pz, sys, {0.0, 0.0}, true, opt, free_field);
    const double t_free = seconds_since(t0);

    const ResidualReport rr = periodicity_residual(pz, sys, a.samples, opt);
    const bool ok = rr.rel() <= 5.0 * a.eps;
    const double a_used = fixed ? aspect(cell) : A;
    const char* path = choose_path(pz, sys.sources.size(), sys.targets.size()) == ApplyPath::Accelerated ? "nufft" : "direct";
    std::printf("%8g %8zu %7s %9.3f %9.3f %9.3f %9.3f %9.3f %11.3e%s\n", a_used, pz.rank(), path, t_build, t_per,
                t_near, t_total, t_free, rr.rel(), ok ? "" : "  FAIL");
    if (!ok) {
      char b[128];
      std::snprintf(b, sizeof b, "A=%g residual %.3e exceeds 5*eps=%.3e", a_used, rr.rel(), 5.0 * a.eps);
      failures.push_back(b);
    }
    std::ostringstream row;
    row << "{\"aspect\": " << jnum(a_used) << ", \"cell\": {\"d\": " << jnum(cell.d) << ", \"xi\": " << jnum(cell.xi)
        << ", \"eta\": " << jnum(cell.eta) << ", \"periodicity\": " << static_cast<int>(cell.periodicity)
        << "}, \"rank\": " << pz.rank() << ", \"path\": " << jstr(path) << ", \"residuals\": {\"e1\": " << jnum(rr.e1)
        << ", \"e2\": " << jnum(rr.e2) << ", \"scale\": " << jnum(rr.scale) << ", \"rel\": " << jnum(rr.rel())
        << "}, \"timings\": {\"build\": " << jnum(t_build) << ", \"per\": " << jnum(t_per) << ", \"near\": "
        << jnum(t_near) << ", \"total\": " << jnum(t_total) << ", \"free\": " << jnum(t_free)
        << "}, \"error\": " << jnum(rr.rel()) << ", \"pass\": " << (ok ? "true" : "false") << "}";
    rows.push_back(row.str());

    if (!a.dump_sources.empty()) {
      std::FILE* f = open_out(a.dump_sources);
      for (std::size_t j = 0; j < sys.sources.size(); ++j) {
        if (is_scalar(pz.pde))
          std::fprintf(f, "%.17g %.17g %.17g\n", sys.sources[j].x, sys.sources[j].y, sys.charges[j]);
        else
          std::fprintf(f, "%.17g %.17g %.17g %.17g\n", sys.sources[j].x, sys.sources[j].y, sys.forces[j].x,
                       sys.forces[j].y);
      }
      std::fclose(f);
    }
    if (!a.dump_fields.empty()) {
      std::FILE* f = open_out(a.dump_fields);
      print_fields(f, sys.targets, total, opt_field.with_pressure);
      std::fclose(f);
    }
  }
  if (!a.out.empty()) {
    std::ofstream o(a.out);
    require(o.good(), ErrorCode::ParseError, a.out + ": cannot open for writing");
    o << "{\"command\": \"validate\", \"pde\": " << jstr(a.pde) << ", \"beta\": " << jnum(a.beta)
      << ", \"eps\": " << jnum(a.eps) << ", \"accel\": " << jstr(a.accel) << ", \"n_src\": " << a.n_src
      << ", \"seed\": " << a.seed << ", \"samples\": " << a.samples << ", \"threads\": " << a.threads
      << ",\n \"rows\": [";
    for (std::size_t i = 0; i < rows.size(); ++i) o << (i ? ",\n  " : "\n  ") << rows[i];
    o << "],\n \"pass\": " << (failures.empty() ? "true" : "false") << ", \"failures\": [";
    for (std::size_t i = 0; i < failures.size(); ++i) o << (i ? ", " : "") << jstr(failures[i]);
    o << "]}\n";
  }
  for (const std::string& f : failures) std::fprintf(stderr, "FAIL: %s\n", f.c_str());
  return failures.empty() ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    require(a.eps >= 1e-13 && a.eps <= 1e-3, ErrorCode::PrecisionOutOfRange, "--eps must lie in [1e-13, 1e-3]");
    return a.cmd == "apply" ? run_apply(a) : run_validate(a);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    return 2;
  } catch (const Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
