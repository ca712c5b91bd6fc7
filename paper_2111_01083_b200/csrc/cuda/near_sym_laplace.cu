// Instantiations of the symmetric near tile: Laplace log tile (SymLaplace, both precision tiers).
#include "near_sym_impl.cuh"

namespace pwb {
namespace sym {

bool launch_laplace(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd, long long* rsh,
                    const SymRange& r) {
  // product form (engine.cu prod_form): binned points scaled to period 2; one image row
  // (singly periodic) or the unskewed 3 x 3 block (doubly periodic)
  if (a.prod_sc != 0.0 && a.lowp && a.nxi == 3 && (a.nrow == 1 || (a.nrow == 3 && a.unskewed))) {
    if (a.nrow == 1) {
      if (a.coarse_log)
        launch_sym_shape<SymLaplace<true, true, true>, 3, 1>(a, st, fx, rsd, rsh, r);
      else
        launch_sym_shape<SymLaplace<true, false, true>, 3, 1>(a, st, fx, rsd, rsh, r);
    } else {
      if (a.coarse_log)
        launch_sym_shape<SymLaplace<true, true, true>, 3, 3, true>(a, st, fx, rsd, rsh, r);
      else
        launch_sym_shape<SymLaplace<true, false, true>, 3, 3, true>(a, st, fx, rsd, rsh, r);
    }
    return true;
  }
  if (a.lowp && a.coarse_log) return dispatch_sym<SymLaplace<true, true>>(a, st, fx, rsd, rsh, r);
  return a.lowp ? dispatch_sym<SymLaplace<true>>(a, st, fx, rsd, rsh, r)
                : dispatch_sym<SymLaplace<false>>(a, st, fx, rsd, rsh, r);
}

}  // namespace sym
}  // namespace pwb
