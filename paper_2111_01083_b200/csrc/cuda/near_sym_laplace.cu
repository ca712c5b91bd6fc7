// Instantiations of the symmetric near tile: Laplace log tile (SymLaplace, both precision tiers).
#include "near_sym_impl.cuh"

namespace pwb {
namespace sym {

bool launch_laplace(const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd, long long* rsh,
                    const SymRange& r) {
  // product form (engine.cu prod_form): binned points, scaled to period 2 when the period is
  // a power of two (prod == 1), unscaled otherwise (prod == 2); one image row (singly
  // periodic) or the unskewed 3 x 3 block (doubly periodic)
  if (a.prod != 0 && a.lowp && a.nxi == 3 && (a.nrow == 1 || (a.nrow == 3 && a.unskewed))) {
    auto go = [&](auto clog, auto prod) {
      using K = SymLaplace<true, decltype(clog)::value, decltype(prod)::value>;
      if (a.nrow == 1)
        launch_sym_shape<K, 3, 1>(a, st, fx, rsd, rsh, r);
      else
        launch_sym_shape<K, 3, 3, true>(a, st, fx, rsd, rsh, r);
    };
    using P1 = std::integral_constant<int, 1>;
    using P2 = std::integral_constant<int, 2>;
    if (a.coarse_log)
      a.prod == 1 ? go(std::true_type{}, P1{}) : go(std::true_type{}, P2{});
    else
      a.prod == 1 ? go(std::false_type{}, P1{}) : go(std::false_type{}, P2{});
    return true;
  }
  if (a.lowp && a.coarse_log) return dispatch_sym<SymLaplace<true, true>>(a, st, fx, rsd, rsh, r);
  return a.lowp ? dispatch_sym<SymLaplace<true>>(a, st, fx, rsd, rsh, r)
                : dispatch_sym<SymLaplace<false>>(a, st, fx, rsd, rsh, r);
}

}  // namespace sym
}  // namespace pwb
