// Symmetric near-image P2P for targets == sources: the host-side entry points, the
// fixed-point readout and the per-kind dispatch. The tile itself (functors, kernel,
// launcher) is in near_sym_impl.cuh, instantiated per family in near_sym_laplace.cu,
// near_sym_modhelm.cu and near_sym_stokes.cu.
#include "near_sym_impl.cuh"

namespace pwb {
namespace {

__global__ void fx_finish_kernel(const unsigned long long* acc, size_t n, double* out0, int nout0, double* out1,
                                 int nout1, const int* out_row) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nout = nout0 + nout1;
  if (i >= n * nout) return;
  const long long a = static_cast<long long>(acc[3 * i]);
  const long long b = static_cast<long long>(acc[3 * i + 1]);
  const long long c = static_cast<long long>(acc[3 * i + 2]);
  const double v = fma(static_cast<double>(a), 0x1p22,
                       fma(static_cast<double>(b), 0x1p-20, static_cast<double>(c) * 0x1p-62));
  const size_t l = out_row ? static_cast<size_t>(out_row[i / nout]) : i / nout;
  const int k = static_cast<int>(i % nout);
  double* dst = k < nout0 ? out0 + l * nout0 + k : out1 + l * nout1 + (k - nout0);
  *dst += v;
}

}  // namespace

void launch_fx_finish(const unsigned long long* fx, size_t n, double* out0, int nout0, double* out1, int nout1,
                      const int* out_row, cudaStream_t st) {
  const size_t total = n * static_cast<size_t>(nout0 + nout1);
  if (total == 0) return;
  fx_finish_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(fx, n, out0, nout0, out1, nout1,
                                                                               out_row);
  count_launches(1);
}

// upper bound on the number of tiles (the smallest tile is 256 points)
size_t near_sym_tiles(size_t n) { return (n + 255) / 256; }

namespace {
template <class K>
long item_count(size_t n) {
  const size_t tile = static_cast<size_t>(sym::kT) * K::TPT;
  const long nb = static_cast<long>((n + tile - 1) / tile);
  long items = 0;
  for (long I = 0; I < nb; ++I) items += (nb - I + K::CHUNK - 1) / K::CHUNK;
  return items;
}
}  // namespace

long near_sym_item_count(NearKind kind, size_t n) {
  switch (kind) {
    case NearKind::Laplace: return item_count<sym::SymLaplace<false>>(n);
    case NearKind::ModHelm: return item_count<sym::SymModHelm<false, false>>(n);
    case NearKind::ModHelmGrad: return item_count<sym::SymModHelm<true, false>>(n);
    case NearKind::Stokes: return item_count<sym::SymStokes<false, false>>(n);
    case NearKind::StokesP: return item_count<sym::SymStokes<true, false>>(n);
    default: return 0;
  }
}

bool near_sym_supported(NearKind kind) {
  return kind == NearKind::Laplace || kind == NearKind::ModHelm || kind == NearKind::ModHelmGrad ||
         kind == NearKind::Stokes || kind == NearKind::StokesP;
}

bool launch_near_sym(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, int* rsd, int* rsh,
                     const SymRange& r) {
  if (a.nt == 0) {
    if (r.total_items) *r.total_items = 0;
    return true;
  }
  // precision tier (pw_math.cuh log_pos_k / k01_tile): reduced when eps allows it
  switch (kind) {
    case NearKind::Laplace: return sym::launch_laplace(a, st, fx, rsd, rsh, r);
    case NearKind::ModHelm:
    case NearKind::ModHelmGrad: return sym::launch_modhelm(kind, a, st, fx, rsd, rsh, r);
    case NearKind::Stokes:
    case NearKind::StokesP: return sym::launch_stokes(kind, a, st, fx, rsd, rsh, r);
    default: return false;
  }
}

}  // namespace pwb
