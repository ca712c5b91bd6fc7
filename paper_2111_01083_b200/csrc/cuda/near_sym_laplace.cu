// Instantiations of the symmetric near tile: Laplace log tile (SymLaplace, both precision tiers).
#include "near_sym_impl.cuh"

namespace pwb {
namespace sym {

bool launch_laplace(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd, long long* rsh,
                    const SymRange& r) {
  if (a.lowp && a.coarse_log) return dispatch_sym<SymLaplace<true, true>>(a, st, fx, rsd, rsh, r);
  return a.lowp ? dispatch_sym<SymLaplace<true>>(a, st, fx, rsd, rsh, r)
                : dispatch_sym<SymLaplace<false>>(a, st, fx, rsd, rsh, r);
}

}  // namespace sym
}  // namespace pwb
