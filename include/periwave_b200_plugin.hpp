// Reference-side plug-in: the B200 near field inside the REFERENCE's own total_field.
//
// Compile this header against the reference's headers (proj/include), not against this
// repo's drop-in periwave.hpp; it talks to the product through the C-ABI only
// (periwave_b200.h), so the reference library and libperiwave_b200.so coexist in one
// process (the product is linked -Bsymbolic: its internal calls never bind to the
// reference's same-named periwave:: symbols, and it exports nothing the reference calls).
//
//   #include "periwave/apply.hpp"            // the reference
//   #include "periwave_b200_plugin.hpp"      // this repo
//   periwave_b200::NearEvaluator gpu;         // one per thread of use (or share: it locks)
//   auto r = periwave::total_field(pz, sys, opt, &gpu);
//
// The override point is FreeSpaceEvaluator::accumulate (proj/include/periwave/apply.hpp:
// 36-45, documented in proj/README.md:133-136); total_field calls it once per near image
// (proj/src/apply.cpp:548-556) and this class forwards each call to pwb_accumulate, which
// adds that image's direct sum on the GPU with the reference's semantics: exact-zero
// (t - s) - shift pairs skipped on the identity image, CoincidentSourceTarget otherwise
// (apply.cpp:531-546), outputs sized like ensure_sizes (apply.cpp:395-405), errors thrown
// as periwave::Error with the reference's codes.
#pragma once

#include <cstddef>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "periwave/apply.hpp"
#include "periwave/errors.hpp"
#include "periwave_b200.h"

namespace periwave_b200 {

class NearEvaluator : public periwave::FreeSpaceEvaluator {
 public:
  explicit NearEvaluator(int device = -1) : device_(device) {}
  ~NearEvaluator() override {
    if (h_) pwb_periodizer_free(h_);
  }
  NearEvaluator(const NearEvaluator&) = delete;
  NearEvaluator& operator=(const NearEvaluator&) = delete;

  void accumulate(const periwave::Periodizer& pz, const periwave::ParticleSystem& sys, periwave::Vec2 shift,
                  bool identity_shift, const periwave::ApplyOptions& opt,
                  periwave::FieldResult& out) const override {
    std::lock_guard<std::mutex> g(mu_);
    const std::size_t ns = sys.sources.size(), nt = sys.targets.size();
    const bool multipole = pz.multipole_order >= 1;
    const bool velocity = !multipole && (pz.pde == periwave::Pde::Stokes || pz.pde == periwave::Pde::ModStokes);
    // the strength lengths of check_strengths (apply.cpp:350-364): the C-ABI sees pointers only
    using periwave::ErrorCode;
    if (multipole)
      periwave::require(sys.coefficients.size() == ns, ErrorCode::LengthMismatch,
                        "multipole apply requires one complex coefficient per source");
    else if (pz.dlp)
      periwave::require(sys.forces.size() == ns && sys.normals.size() == ns, ErrorCode::LengthMismatch,
                        "double-layer apply requires a force vector and a unit normal per source");
    else if (velocity)
      periwave::require(sys.forces.size() == ns, ErrorCode::LengthMismatch,
                        "velocity apply requires one force vector per source");
    else
      periwave::require(sys.charges.size() == ns, ErrorCode::LengthMismatch,
                        "scalar apply requires one charge per source");
    pwb_periodizer* h = handle(pz);
    // ensure_sizes (apply.cpp:395-405): resize only when the length differs
    auto fit = [nt](auto& v) {
      if (v.size() != nt) v.assign(nt, typename std::decay_t<decltype(v)>::value_type{});
    };
    pwb_field f{};
    f.memory = PWB_MEM_HOST;
    if (multipole) {
      fit(out.complex_scalar);
      f.complex_scalar = reinterpret_cast<double*>(out.complex_scalar.data());
    } else if (velocity) {
      fit(out.velocity);
      f.velocity = reinterpret_cast<double*>(out.velocity.data());
      if (opt.with_pressure) {
        fit(out.pressure);
        f.pressure = out.pressure.data();
      }
    } else {
      fit(out.scalar);
      f.scalar = out.scalar.data();
    }
    // Vec2 / cplx are two contiguous doubles in the reference too: no copies. data() of an
    // empty vector may be null; the C-ABI accepts that when the count is zero.
    pwb_system s{};
    s.n_src = ns;
    s.n_tgt = nt;
    s.sources = reinterpret_cast<const double*>(sys.sources.data());
    s.targets = reinterpret_cast<const double*>(sys.targets.data());
    s.charges = sys.charges.empty() ? nullptr : sys.charges.data();
    s.forces = sys.forces.empty() ? nullptr : reinterpret_cast<const double*>(sys.forces.data());
    s.normals = sys.normals.empty() ? nullptr : reinterpret_cast<const double*>(sys.normals.data());
    s.coefficients = sys.coefficients.empty() ? nullptr : reinterpret_cast<const double*>(sys.coefficients.data());
    s.memory = PWB_MEM_HOST;
    pwb_options o;
    pwb_options_default(&o);
    o.path = static_cast<int>(opt.path);
    o.threads = opt.threads;
    o.with_pressure = opt.with_pressure ? 1 : 0;
    o.nufft_eps = opt.nufft_eps;
    o.device = device_;
    const int rc = pwb_accumulate(h, &s, shift.x, shift.y, identity_shift ? 1 : 0, &o, &f);
    ++calls_;
    if (rc == PWB_OK) return;
    if (rc >= 1 && rc <= 19) throw periwave::Error(static_cast<periwave::ErrorCode>(rc - 1), pwb_last_error());
    throw std::runtime_error(std::string("periwave-b200: ") + pwb_last_error());
  }

  // accumulate calls served (the reference's Counting test pattern, test_apply.cpp:337-357)
  int calls() const {
    std::lock_guard<std::mutex> g(mu_);
    return calls_;
  }

 private:
  // A product periodizer for the near sum, rebuilt only when the periodizer changes: the
  // direct image sums need (pde, beta, cell, dlp, multipole order), not the far tables.
  pwb_periodizer* handle(const periwave::Periodizer& pz) const {
    const Key k{static_cast<int>(pz.pde), pz.beta, pz.cell.d, pz.cell.xi, pz.cell.eta,
                static_cast<int>(pz.cell.periodicity), pz.cell.m0, pz.eps, pz.dlp, pz.multipole_order};
    if (h_ && k == key_) return h_;
    if (h_) pwb_periodizer_free(h_);
    h_ = nullptr;
    pwb_cell c;
    const int rc0 = pwb_make_unit_cell(pz.cell.d, pz.cell.xi, pz.cell.eta,
                                       pz.cell.periodicity == periwave::Periodicity::Singly ? PWB_SINGLY : PWB_DOUBLY,
                                       &c);
    if (rc0 != PWB_OK) throw std::runtime_error(std::string("periwave-b200: ") + pwb_last_error());
    pwb_periodizer* h = nullptr;
    const int rc = pwb_periodizer_new(static_cast<int>(pz.pde), pz.beta, &c, pz.eps, pz.dlp ? 1 : 0,
                                      pz.multipole_order, pz.requires_neutrality ? 1 : 0, &h);
    if (rc != PWB_OK) throw std::runtime_error(std::string("periwave-b200: ") + pwb_last_error());
    h_ = h;
    key_ = k;
    return h_;
  }

  struct Key {
    int pde;
    double beta, d, xi, eta;
    int per, m0;
    double eps;
    bool dlp;
    int order;
    bool operator==(const Key& o) const {
      return pde == o.pde && beta == o.beta && d == o.d && xi == o.xi && eta == o.eta && per == o.per &&
             m0 == o.m0 && eps == o.eps && dlp == o.dlp && order == o.order;
    }
  };
  int device_;
  mutable std::mutex mu_;
  mutable pwb_periodizer* h_ = nullptr;
  mutable Key key_{};
  mutable int calls_ = 0;
};

}  // namespace periwave_b200
