// Drop-in check and timer: the reference's own call shape against the C-ABI fast path.
//
//   pwb-dropin-bench PDE BETA D XI ETA PERIODICITY EPS INPUTS.bin OUT_PREFIX [REPS]
//
// INPUTS.bin: uint64 n, uint64 w (1 = charges, 2 = forces), 2n doubles sources, w*n
// doubles strengths. Targets = sources.
//
// (1) periwave::total_field(pz, sys) exactly as a reference user calls it
//     (proj/include/periwave/apply.hpp:58-60): a fresh ParticleSystem whose `targets` is a
//     separate std::vector holding a copy of `sources` (cell.hpp:58-65), the periodizer by
//     const&, host vectors in and out. Timed per call (wall clock, host to host).
// (2) pwb_total_field through the C-ABI with targets == sources (one host pointer), the
//     path the headline bench line takes with host buffers.
// Writes OUT_PREFIX.dropin.bin / OUT_PREFIX.capi.bin (the output doubles) and prints one
// JSON line with the per-call times. The first call of each arm is the warm-up (plan
// upload) and is reported apart.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "periwave/periwave.hpp"
#include "periwave_b200.h"

namespace {

double now_ms() {
  using C = std::chrono::steady_clock;
  return std::chrono::duration<double, std::milli>(C::now().time_since_epoch()).count();
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : v[v.size() / 2];
}

void write(const std::string& path, const double* p, size_t n) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f || std::fwrite(p, sizeof(double), n, f) != n) {
    std::fprintf(stderr, "cannot write %s\n", path.c_str());
    std::exit(3);
  }
  std::fclose(f);
}

std::string list(const std::vector<double>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
  return s + "]";
}

}  // namespace

// --cache-check: the drop-in API's per-periodizer plan cache (api.cu PlanCache, 8 entries)
// under eviction. 12 distinct periodizers (3 cell heights x 4 eps) are applied round-robin three
// times to a small system; every result must equal, bitwise, the first result of the same
// periodizer (a rebuilt plan after eviction is the same deterministic computation), and a
// periodizer copied by value must hit the same plan. Prints one JSON line; exit 1 on mismatch.
int cache_check() {
  periwave::Rng rng(77);
  const size_t n = 300;
  periwave::ParticleSystem sys;
  sys.sources.resize(n);
  sys.charges.resize(n);
  double mean = 0.0;
  for (size_t i = 0; i < n; ++i) {
    sys.sources[i] = {rng.uniform() - 0.5, 0.8 * (rng.uniform() - 0.5)};
    mean += (sys.charges[i] = rng.uniform() - 0.5);
  }
  for (auto& q : sys.charges) q -= mean / n;
  sys.targets = sys.sources;
  std::vector<periwave::Periodizer> pzs;
  for (double eta : {0.8, 0.9, 1.0})  // |y| <= 0.4: the points lie in all three cells (d >= |e2|)
    for (double eps : {1e-6, 1e-8, 1e-10, 1e-12})
      pzs.push_back(periwave::make_periodizer(periwave::Pde::Poisson, 0.0,
                                              periwave::make_unit_cell(1.0, 0.0, eta, periwave::Periodicity::Doubly), eps));
  std::vector<std::vector<double>> first(pzs.size());
  int mismatches = 0, calls = 0;
  for (int round = 0; round < 3; ++round)
    for (size_t k = 0; k < pzs.size(); ++k) {
      const periwave::Periodizer copy = pzs[k];  // equal content, distinct object
      const periwave::FieldResult r = periwave::total_field(round == 1 ? copy : pzs[k], sys);
      ++calls;
      if (round == 0)
        first[k] = r.scalar;
      else if (r.scalar != first[k])
        ++mismatches;
    }
  std::printf("{\"cache_check\": true, \"periodizers\": %zu, \"calls\": %d, \"mismatches\": %d}\n", pzs.size(), calls,
              mismatches);
  return mismatches ? 1 : 0;
}

// --error-check: the drop-in total_field / apply_far leave the point checks to the device
// (api.cu validated_device_call); the error a caller sees must still be the one the
// reference raises first (validate_system before every other check, apply.cpp:417-430,
// cell.cpp:77-94). Prints one JSON line; exit 1 when a case raises something else.
int error_check() {
  using periwave::ErrorCode;
  periwave::Rng rng(5);
  const size_t n = 400;
  periwave::ParticleSystem good;
  good.sources.resize(n);
  good.charges.resize(n);
  double mean = 0.0;
  for (size_t i = 0; i < n; ++i) {
    good.sources[i] = {rng.uniform() - 0.5, rng.uniform() - 0.5};
    mean += (good.charges[i] = rng.uniform() - 0.5);
  }
  for (auto& q : good.charges) q -= mean / n;
  good.targets = good.sources;
  const periwave::Periodizer pz = periwave::make_periodizer(
      periwave::Pde::Poisson, 0.0, periwave::make_unit_cell(1.0, 0.0, 1.0, periwave::Periodicity::Doubly), 1e-8);
  int failures = 0, cases = 0;
  std::string report;
  auto expect = [&](const char* name, const periwave::ParticleSystem& sys, int want, bool far_only) {
    int got = -1;  // -1: no error
    try {
      if (far_only)
        periwave::apply_far(pz, sys);
      else
        periwave::total_field(pz, sys);
    } catch (const periwave::Error& e) {
      got = static_cast<int>(e.code());
    }
    ++cases;
    if (got != want) ++failures;
    report += std::string(report.empty() ? "" : ", ") + "\"" + name + "\": " + std::to_string(got);
  };
  for (bool far_only : {false, true}) {
    const std::string tag = far_only ? "far_" : "";
    expect((tag + "ok").c_str(), good, -1, far_only);
    periwave::ParticleSystem s = good;
    s.sources[7].x = 0.75;  // outside the cell
    expect((tag + "outside_source").c_str(), s, static_cast<int>(ErrorCode::OutOfInterval), far_only);
    s = good;
    s.targets[9].y = -0.9;
    expect((tag + "outside_target").c_str(), s, static_cast<int>(ErrorCode::OutOfInterval), far_only);
    s = good;
    s.charges.pop_back();
    expect((tag + "short_charges").c_str(), s, static_cast<int>(ErrorCode::LengthMismatch), far_only);
    s.sources[3].x = 2.0;  // points are checked before lengths
    expect((tag + "outside_and_short").c_str(), s, static_cast<int>(ErrorCode::OutOfInterval), far_only);
    s = good;
    s.charges[0] += 1.0;
    expect((tag + "not_neutral").c_str(), s, static_cast<int>(ErrorCode::NotNeutral), far_only);
    s.targets[1].x = -3.0;  // ... and before neutrality
    expect((tag + "outside_and_not_neutral").c_str(), s, static_cast<int>(ErrorCode::OutOfInterval), far_only);
  }
  std::printf("{\"error_check\": true, \"cases\": %d, \"failures\": %d, \"codes\": {%s}}\n", cases, failures,
              report.c_str());
  return failures ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc == 2 && std::string(argv[1]) == "--error-check") {
    try {
      return error_check();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  if (argc == 2 && std::string(argv[1]) == "--cache-check") {
    try {
      return cache_check();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  if (argc < 10) {
    std::fprintf(stderr, "usage: %s PDE BETA D XI ETA PERIODICITY EPS INPUTS.bin OUT_PREFIX [REPS]\n", argv[0]);
    return 2;
  }
  const int pde = std::atoi(argv[1]);
  const double beta = std::atof(argv[2]), d = std::atof(argv[3]), xi = std::atof(argv[4]), eta = std::atof(argv[5]);
  const int per = std::atoi(argv[6]);
  const double eps = std::atof(argv[7]);
  const std::string out_prefix = argv[9];
  const int reps = argc > 10 ? std::atoi(argv[10]) : 5;

  FILE* f = std::fopen(argv[8], "rb");
  uint64_t hdr[2];
  if (!f || std::fread(hdr, sizeof(uint64_t), 2, f) != 2) {
    std::fprintf(stderr, "cannot read %s\n", argv[8]);
    return 2;
  }
  const size_t n = hdr[0], w = hdr[1];
  std::vector<double> pts(2 * n), str(w * n);
  if (std::fread(pts.data(), sizeof(double), pts.size(), f) != pts.size() ||
      std::fread(str.data(), sizeof(double), str.size(), f) != str.size()) {
    std::fprintf(stderr, "short read %s\n", argv[8]);
    return 2;
  }
  std::fclose(f);

  try {
    // ---- (1) the reference's call shape
    const periwave::UnitCell cell =
        periwave::make_unit_cell(d, xi, eta, per == 1 ? periwave::Periodicity::Singly : periwave::Periodicity::Doubly);
    const periwave::Periodizer pz = periwave::make_periodizer(static_cast<periwave::Pde>(pde), beta, cell, eps);
    std::vector<double> dropin_ms;
    periwave::FieldResult res;
    for (int r = 0; r <= reps; ++r) {
      periwave::ParticleSystem sys;  // rebuilt per call, as a caller with fresh data would
      sys.sources.resize(n);
      for (size_t i = 0; i < n; ++i) sys.sources[i] = {pts[2 * i], pts[2 * i + 1]};
      if (w == 1) {
        sys.charges = str;
      } else {
        sys.forces.resize(n);
        for (size_t i = 0; i < n; ++i) sys.forces[i] = {str[2 * i], str[2 * i + 1]};
      }
      sys.targets = sys.sources;  // a separate vector: equal bytes, distinct storage
      const double t0 = now_ms();
      res = periwave::total_field(pz, sys);
      dropin_ms.push_back(now_ms() - t0);
    }
    const bool vel = !res.velocity.empty();
    const size_t nout = vel ? 2 * n : n;
    write(out_prefix + ".dropin.bin", vel ? reinterpret_cast<const double*>(res.velocity.data()) : res.scalar.data(),
          nout);

    // ---- (2) the C-ABI with one host array for sources and targets
    pwb_cell c;
    if (pwb_make_unit_cell(d, xi, eta, per, &c) != PWB_OK) throw std::runtime_error(pwb_last_error());
    pwb_periodizer* h = nullptr;
    if (pwb_make_periodizer(pde, beta, &c, eps, &h) != PWB_OK) throw std::runtime_error(pwb_last_error());
    pwb_system s{};
    s.n_src = s.n_tgt = n;
    s.sources = s.targets = pts.data();
    (w == 1 ? s.charges : s.forces) = str.data();
    s.memory = PWB_MEM_HOST;
    pwb_options o;
    pwb_options_default(&o);
    std::vector<double> out(nout);
    pwb_field fo{};
    (vel ? fo.velocity : fo.scalar) = out.data();
    fo.memory = PWB_MEM_HOST;
    std::vector<double> capi_ms;
    for (int r = 0; r <= reps; ++r) {
      const double t0 = now_ms();
      if (pwb_total_field(h, &s, &o, &fo) != PWB_OK) throw std::runtime_error(pwb_last_error());
      capi_ms.push_back(now_ms() - t0);
    }
    write(out_prefix + ".capi.bin", out.data(), nout);
    pwb_periodizer_free(h);

    const double first_dropin = dropin_ms.front(), first_capi = capi_ms.front();
    dropin_ms.erase(dropin_ms.begin());
    capi_ms.erase(capi_ms.begin());
    std::printf(
        "{\"n\": %zu, \"reps\": %d, \"dropin_ms\": %s, \"capi_ms\": %s, \"dropin_median_ms\": %.3f, "
        "\"capi_median_ms\": %.3f, \"dropin_first_ms\": %.3f, \"capi_first_ms\": %.3f}\n",
        n, reps, list(dropin_ms).c_str(), list(capi_ms).c_str(), median(dropin_ms), median(capi_ms), first_dropin,
        first_capi);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
