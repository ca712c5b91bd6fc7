// Instantiations of the symmetric near tile: modified-Helmholtz tiles (SymModHelm, with / without gradient, both tiers).
#include "near_sym_impl.cuh"

namespace pwb {
namespace sym {

bool launch_modhelm(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd,
                    long long* rsh, const SymRange& r) {
  // a.lowp: 0 full tier, 1 reduced (eps >= 1e-11), 2 coarse Bessel (eps >= 1e-9)
  if (kind == NearKind::ModHelmGrad)
    return a.lowp == 2 ? dispatch_sym<SymModHelm<true, true, true>>(a, st, fx, rsd, rsh, r)
           : a.lowp    ? dispatch_sym<SymModHelm<true, true>>(a, st, fx, rsd, rsh, r)
                       : dispatch_sym<SymModHelm<true, false>>(a, st, fx, rsd, rsh, r);
  return a.lowp == 2 ? dispatch_sym<SymModHelm<false, true, true>>(a, st, fx, rsd, rsh, r)
         : a.lowp    ? dispatch_sym<SymModHelm<false, true>>(a, st, fx, rsd, rsh, r)
                     : dispatch_sym<SymModHelm<false, false>>(a, st, fx, rsd, rsh, r);
}

}  // namespace sym
}  // namespace pwb
