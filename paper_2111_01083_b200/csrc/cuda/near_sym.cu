// Symmetric near-image P2P for targets == sources: the host-side entry points, the
// fixed-point readout and the per-kind dispatch. The tile itself (functors, kernel,
// launcher) is in near_sym_impl.cuh, instantiated per family in near_sym_laplace.cu,
// near_sym_modhelm.cu and near_sym_stokes.cu.
#include "near_sym_impl.cuh"

#include <cub/device/device_scan.cuh>

#include <mutex>
#include <set>
#include <utility>

namespace pwb {
namespace {

__global__ void fx_finish_kernel(const unsigned long long* acc, size_t n, double* out0, int nout0, double* out1,
                                 int nout1, const int* out_row, const unsigned* maxhi, size_t n_src, int k_host,
                                 const int* flag) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nout = nout0 + nout1;
  if (i >= n * nout) return;
  if (flag && (*flag & 2)) return;  // fixed-point range exceeded: the engine redoes the near field in fp64
  const double inv = fx_scale(-(maxhi ? fx_exponent(*maxhi, n_src) : k_host));
  const long long a = static_cast<long long>(acc[3 * i]);
  const long long b = static_cast<long long>(acc[3 * i + 1]);
  const long long c = static_cast<long long>(acc[3 * i + 2]);
  const double v = fma(static_cast<double>(a), 0x1p22,
                       fma(static_cast<double>(b), 0x1p-20, static_cast<double>(c) * 0x1p-62));
  const size_t l = out_row ? static_cast<size_t>(out_row[i / nout]) : i / nout;
  const int k = static_cast<int>(i % nout);
  double* dst = k < nout0 ? out0 + l * nout0 + k : out1 + l * nout1 + (k - nout0);
  *dst += v * inv;  // exact power-of-two rescale
}

// high word of max |w| over the strengths (q, or both force components); the high
// words of non-negative doubles order like the values, so an integer atomicMax is an
// exact, order-independent max (NaN / inf land above 0x7ff00000)
__global__ void fx_maxhi_kernel(const double* q, const double2* vec, size_t n, unsigned* maxhi) {
  unsigned m = 0u;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
    if (q) m = max(m, static_cast<unsigned>(__double2hiint(q[j])) & 0x7fffffffu);
    if (vec) {
      const double2 f = vec[j];
      m = max(m, static_cast<unsigned>(__double2hiint(f.x)) & 0x7fffffffu);
      m = max(m, static_cast<unsigned>(__double2hiint(f.y)) & 0x7fffffffu);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(maxhi, m);
}

}  // namespace

void launch_fx_finish(const unsigned long long* fx, size_t n, double* out0, int nout0, double* out1, int nout1,
                      const int* out_row, const unsigned* maxhi_dev, size_t n_src, int k_host, const int* flag,
                      cudaStream_t st) {
  const size_t total = n * static_cast<size_t>(nout0 + nout1);
  if (total == 0) return;
  fx_finish_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(fx, n, out0, nout0, out1, nout1,
                                                                               out_row, maxhi_dev, n_src, k_host, flag);
  count_launches(1);
}

void launch_fx_maxhi(const NearArgs& a, unsigned* maxhi, cudaStream_t st) {
  cuda_check(cudaMemsetAsync(maxhi, 0, sizeof(unsigned), st), "memset maxhi");
  if (a.ns == 0) return;
  const size_t blocks = std::min<size_t>((a.ns + 255) / 256, 4 * 148);
  fx_maxhi_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a.q, a.vec, a.ns, maxhi);
  count_launches(1);
}

void set_max_carveout(const void* kernel) {
  // Static shared memory (tile + per-warp column partials) is what limits residency next
  // to registers: ask for the maximum carveout so registers decide (ncu r1: the default
  // carveout capped SymLaplace at 5 blocks on shared memory alone). Per device: a second
  // device in the same process gets its own attribute call.
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "get device");
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert({dev, kernel}).second) return;
  cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared),
             "smem carveout");
}

// upper bound on the number of row tiles (the smallest row tile is 128 points)
size_t near_sym_tiles(size_t n) { return (n + 127) / 128; }

namespace {
template <class K>
long item_count(size_t n) {
  const size_t tile = static_cast<size_t>(K::THREADS) * K::TPT, ct = static_cast<size_t>(sym::kColUnit) * K::CPT;
  const long nb = static_cast<long>((n + tile - 1) / tile), ncb = static_cast<long>((n + ct - 1) / ct);
  const long r = static_cast<long>(tile / ct);
  long items = 0;
  for (long I = 0; I < nb; ++I) items += (ncb - I * r + K::CHUNK - 1) / K::CHUNK;
  return items;
}
// ---- cost-balanced item ranges for the multi-GPU split of the screened tiles ----------
// Bounding box (xmin, -xmax, ymin, -ymax) of every tile; one warp per tile.
__global__ void tile_box_kernel(const double2* __restrict__ p, size_t n, int tile, int nb, double* __restrict__ box) {
  const int t = static_cast<int>((static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= nb) return;
  double b[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  const size_t j0 = static_cast<size_t>(t) * tile;
  for (int i = lane; i < tile; i += 32) {
    const size_t j = j0 + i;
    if (j >= n) break;
    const double2 q = p[j];
    b[0] = fmin(b[0], q.x);
    b[1] = fmin(b[1], -q.x);
    b[2] = fmin(b[2], q.y);
    b[3] = fmin(b[3], -q.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 4; ++c) b[c] = fmin(b[c], __shfl_xor_sync(0xffffffffu, b[c], o));
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 4; ++c) box[4 * static_cast<size_t>(t) + c] = b[c];
}

// Estimated cost of every work item (row tile I, column tiles J0..J1): per tile pair a
// staging overhead plus, per image, what the tile will do with it (near_sym_impl.cuh):
// nothing when masked, a branch-free regime sweep, or the per-pair dispatch.
__global__ void item_cost_kernel(const double* __restrict__ box, const long long* __restrict__ row_start, int nb, int chunk,
                                 long items, const NearArgs a, float* __restrict__ cost) {
  const long item = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= items) return;
  int lo = 0, hi = nb;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (row_start[mid] <= item)
      lo = mid;
    else
      hi = mid;
  }
  const int I = lo;
  const int J0 = I + static_cast<int>(item - row_start[I]) * chunk;
  const int J1 = min(nb, J0 + chunk);
  double rb[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) rb[c] = box[4 * static_cast<size_t>(I) + c];
  float c_item = 0.0f;
  for (int J = J0; J < J1; ++J) {
    double cb[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) cb[c] = box[4 * static_cast<size_t>(J) + c];
    float c_pair = 0.25f;  // staging, boxes, column flush
    for (int img = 0; img < a.nxi * a.nrow; ++img) {
      double xl, xh;
      image_xrange(rb, cb, a.shx[img], a.shy[img / a.nxi], a.beta2, xl, xh);
      if (xl * 0.9999 >= a.xcut2) continue;
      // relative costs calibrated on c5 at N = 1e6 (tools/shard_balance.py, 8 ranks:
      // max/mean 1.14 -> 1.09 -> 1.04 -> 1.025 over three settings): a branch-free regime
      // sweep 1, the per-pair dispatch 3.6 (regime-divergent warps, no cross-source
      // interleave; all-series 3.0), the diagonal tile's careful image-inner path 7
      float ci;
      if (J == I)
        ci = 7.0f;
      else if (const int reg = pwk::regime_of(xl, xh, a.xcut2))
        ci = reg == 2 ? 1.0f : 1.1f;
      else
        ci = xh * 1.0001 < 4.0 ? 3.0f : 3.6f;
      c_pair += ci;
    }
    c_item += c_pair;
  }
  cost[item] = c_item;
}

// bounds[r] = first item whose inclusive cost prefix exceeds r / world of the total
__global__ void split_kernel(const float* __restrict__ prefix, long items, int world, long* __restrict__ bounds) {
  const int r = threadIdx.x;
  if (r > world) return;
  if (r == 0 || r == world) {
    bounds[r] = r == 0 ? 0 : items;
    return;
  }
  const double target = static_cast<double>(prefix[items - 1]) * r / world;
  long lo = 0, hi = items;  // first index with prefix > target
  while (lo < hi) {
    const long mid = (lo + hi) >> 1;
    if (static_cast<double>(prefix[mid]) > target)
      hi = mid;
    else
      lo = mid + 1;
  }
  bounds[r] = lo;
}

}  // namespace

void near_sym_shape(NearKind kind, int* tile, int* chunk) {
  auto set = [&](auto k) {
    using K = decltype(k);
    static_assert(K::CPT == K::TPT || !K::CULL, "the cost split assumes square tiles");
    *tile = K::THREADS * K::TPT;
    *chunk = K::CHUNK;
  };
  switch (kind) {
    case NearKind::Laplace: set(sym::SymLaplace<false>{}); break;
    case NearKind::ModHelm: set(sym::SymModHelm<false, false>{}); break;
    case NearKind::ModHelmGrad: set(sym::SymModHelm<true, false>{}); break;
    case NearKind::Stokes: set(sym::SymStokes<false, false>{}); break;
    case NearKind::StokesP: set(sym::SymStokes<true, false>{}); break;
    default: *tile = 0; *chunk = 0;
  }
}

size_t near_sym_split_bytes(size_t n, long items) {
  size_t tmp = 0;
  cuda_check(cub::DeviceScan::InclusiveSum(nullptr, tmp, static_cast<const float*>(nullptr), static_cast<float*>(nullptr),
                                           static_cast<long long>(items > 0 ? items : 1)),
             "scan size");
  const size_t nb = near_sym_tiles(n);
  return 4 * nb * sizeof(double) + 2 * static_cast<size_t>(items) * sizeof(float) + tmp + 65 * sizeof(long) + 6 * 256;
}

void near_sym_split(NearKind kind, const NearArgs& a, int world, long* bounds_host, void* ws, size_t ws_bytes,
                    long long* row_start_dev, long long* row_start_host, cudaStream_t st) {
  int tile = 0, chunk = 0;
  near_sym_shape(kind, &tile, &chunk);
  const int nb = static_cast<int>((a.nt + tile - 1) / tile);
  long items = 0;
  for (int I = 0; I < nb; ++I) {
    row_start_host[I] = items;
    items += (nb - I + chunk - 1) / chunk;
  }
  row_start_host[nb] = items;
  auto align = [](size_t v) { return (v + 255) & ~static_cast<size_t>(255); };
  char* base = static_cast<char*>(ws);
  double* box = reinterpret_cast<double*>(base);
  size_t off = align(4 * static_cast<size_t>(nb) * sizeof(double));
  float* cost = reinterpret_cast<float*>(base + off);
  off += align(static_cast<size_t>(items) * sizeof(float));
  float* prefix = reinterpret_cast<float*>(base + off);
  off += align(static_cast<size_t>(items) * sizeof(float));
  long* bounds = reinterpret_cast<long*>(base + off);
  off += align(65 * sizeof(long));
  if (off > ws_bytes || world > 64) throw_internal("near_sym_split: workspace");
  size_t tmp = ws_bytes - off;
  cuda_check(cudaMemcpyAsync(row_start_dev, row_start_host, (nb + 1) * sizeof(long long), cudaMemcpyHostToDevice, st),
             "row starts");
  tile_box_kernel<<<static_cast<unsigned>((static_cast<size_t>(nb) * 32 + 255) / 256), 256, 0, st>>>(a.tgt, a.nt, tile,
                                                                                                    nb, box);
  item_cost_kernel<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(box, row_start_dev, nb, chunk, items,
                                                                                a, cost);
  cuda_check(cub::DeviceScan::InclusiveSum(base + off, tmp, cost, prefix, static_cast<long long>(items), st), "scan");
  split_kernel<<<1, 128, 0, st>>>(prefix, items, world, bounds);
  count_launches(3);
  cuda_check(cudaMemcpyAsync(bounds_host, bounds, (world + 1) * sizeof(long), cudaMemcpyDeviceToHost, st), "D2H bounds");
  cuda_check(cudaStreamSynchronize(st), "split sync");
}

long near_sym_item_count(NearKind kind, size_t n, bool prod) {
  switch (kind) {
    case NearKind::Laplace:  // the product-form tile has its own row tile (near_sym_impl.cuh)
      return prod ? item_count<sym::SymLaplace<true, true, 1>>(n) : item_count<sym::SymLaplace<false>>(n);
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

bool launch_near_sym(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx, long long* rsd,
                     long long* rsh, const SymRange& r) {
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
