// Instantiations of the symmetric near tile: Stokeslet tiles (SymStokes, with / without pressure, both tiers).
#include "near_sym_impl.cuh"

namespace pwb {
namespace sym {

bool launch_stokes(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd,
                   long long* rsh, const SymRange& r) {
  if (kind == NearKind::StokesP)
    return a.lowp ? dispatch_sym<SymStokes<true, true>>(a, st, fx, rsd, rsh, r)
                  : dispatch_sym<SymStokes<true, false>>(a, st, fx, rsd, rsh, r);
  // product form (engine.cu prod_form): binned points (scaled to period 2 when the period is
  // a power of two, prod == 1; unscaled otherwise, prod == 2), unskewed 3 x 3 images
  if (a.prod != 0 && a.lowp && a.nxi == 3 && a.nrow == 3 && a.unskewed) {
    if (a.coarse_log) {
      if (a.prod == 1)
        launch_sym_shape<SymStokes<false, true, true, 1>, 3, 3, true>(a, st, fx, rsd, rsh, r);
      else
        launch_sym_shape<SymStokes<false, true, true, 2>, 3, 3, true>(a, st, fx, rsd, rsh, r);
    } else {
      if (a.prod == 1)
        launch_sym_shape<SymStokes<false, true, false, 1>, 3, 3, true>(a, st, fx, rsd, rsh, r);
      else
        launch_sym_shape<SymStokes<false, true, false, 2>, 3, 3, true>(a, st, fx, rsd, rsh, r);
    }
    return true;
  }
  if (a.lowp && a.coarse_log) return dispatch_sym<SymStokes<false, true, true>>(a, st, fx, rsd, rsh, r);
  return a.lowp ? dispatch_sym<SymStokes<false, true>>(a, st, fx, rsd, rsh, r)
                : dispatch_sym<SymStokes<false, false>>(a, st, fx, rsd, rsh, r);
}

}  // namespace sym
}  // namespace pwb
