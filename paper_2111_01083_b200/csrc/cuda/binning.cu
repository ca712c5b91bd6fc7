// Spatial binning of points before the near tile (Morton order on a uniform grid
// over the cell's bounding box).
//
// The screened kernels (K0 / K1 / K_l) branch per pair: ascending series for
// beta*r <= 2, exponential asymptotics above, skip beyond beta*r = 64
// (pw_math.cuh). With points in generator order every warp sees all three
// regimes and executes every branch; binned, a warp's targets and a source tile
// are each spatially compact, so the branch is warp-uniform except at regime
// boundaries (measured: c5 slice 1498 -> 700 ms, c2 1844 -> 1637 ms;
// tools/sort_experiment.py). The reference has no such step (its per-image
// loops are scalar, apply.cpp:532-540); the permutation changes only the order
// of the fp64 source sums, and outputs land at their original indices.
#include <cub/device/device_radix_sort.cuh>

#include "pw_engine.cuh"

namespace pwb {
namespace {

__device__ __forceinline__ unsigned spread_bits(unsigned v) {  // 16 bits -> even bit positions
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__global__ void morton_key_kernel(const double2* __restrict__ p, size_t n, double x0, double y0, double inv_h,
                                  unsigned* __restrict__ key, int* __restrict__ idx) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 q = p[i];
  const double gx = fmin(fmax((q.x - x0) * inv_h, 0.0), 65535.0);
  const double gy = fmin(fmax((q.y - y0) * inv_h, 0.0), 65535.0);
  key[i] = spread_bits(static_cast<unsigned>(gx)) | (spread_bits(static_cast<unsigned>(gy)) << 1);
  idx[i] = static_cast<int>(i);
}

template <class T>
__global__ void gather_kernel(const T* __restrict__ in, const int* __restrict__ perm, size_t n, T* __restrict__ out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[perm[i]];
}

__global__ void gather_scale_kernel(const double2* __restrict__ in, const int* __restrict__ perm, size_t n, double sc,
                                    double2* __restrict__ out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = in[perm[i]];
  out[i] = make_double2(p.x * sc, p.y * sc);
}

unsigned blocks_for(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

// out[perm[i] * w + k] += in[i * w + k]: sorted-order fixed-point rows back to input order
// (integer adds: exact; perm is a permutation, so no two threads touch the same row)
__global__ void scatter_add_rows_kernel(const unsigned long long* __restrict__ in, const int* __restrict__ perm,
                                        size_t n, int w, unsigned long long* __restrict__ out) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * static_cast<size_t>(w)) return;
  const size_t row = i / w;
  out[static_cast<size_t>(perm[row]) * w + (i - row * w)] += in[i];
}

}  // namespace

size_t morton_order_bytes(size_t n) {
  size_t tmp = 0;
  cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tmp, static_cast<const unsigned*>(nullptr),
                                             static_cast<unsigned*>(nullptr), static_cast<const int*>(nullptr),
                                             static_cast<int*>(nullptr), static_cast<int>(n)),
             "radix sort size");
  // keys in/out + indices in + alignment slack
  return tmp + 2 * n * sizeof(unsigned) + n * sizeof(int) + 4 * 256;
}

void morton_order(const double2* pts, size_t n, const BinBox& box, int* perm, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  if (n == 0) return;
  auto align = [](size_t v) { return (v + 255) & ~static_cast<size_t>(255); };
  char* base = static_cast<char*>(ws);
  unsigned* key_in = reinterpret_cast<unsigned*>(base);
  size_t off = align(n * sizeof(unsigned));
  unsigned* key_out = reinterpret_cast<unsigned*>(base + off);
  off += align(n * sizeof(unsigned));
  int* idx_in = reinterpret_cast<int*>(base + off);
  off += align(n * sizeof(int));
  if (off > ws_bytes) throw_internal("morton_order: workspace too small");
  size_t tmp = ws_bytes - off;
  morton_key_kernel<<<blocks_for(n), 256, 0, st>>>(pts, n, box.x0, box.y0, box.inv_h, key_in, idx_in);
  cuda_check(cub::DeviceRadixSort::SortPairs(base + off, tmp, key_in, key_out, idx_in, perm, static_cast<int>(n), 0,
                                             32, st),
             "radix sort");
  count_launches(1);  // the key kernel (cub's sort passes are library kernels)
}

void gather_double(const double* in, const int* perm, size_t n, double* out, cudaStream_t st) {
  if (n == 0 || in == nullptr) return;
  gather_kernel<double><<<blocks_for(n), 256, 0, st>>>(in, perm, n, out);
  count_launches(1);
}

void scatter_add_rows(const unsigned long long* in, const int* perm, size_t n, int width, unsigned long long* out,
                      cudaStream_t st) {
  if (n == 0) return;
  scatter_add_rows_kernel<<<blocks_for(n * width), 256, 0, st>>>(in, perm, n, width, out);
  count_launches(1);
}

void gather_double2(const double2* in, const int* perm, size_t n, double2* out, cudaStream_t st) {
  if (n == 0 || in == nullptr) return;
  gather_kernel<double2><<<blocks_for(n), 256, 0, st>>>(in, perm, n, out);
  count_launches(1);
}

void gather_scale_double2(const double2* in, const int* perm, size_t n, double sc, double2* out, cudaStream_t st) {
  if (n == 0 || in == nullptr) return;
  gather_scale_kernel<<<blocks_for(n), 256, 0, st>>>(in, perm, n, sc, out);
  count_launches(1);
}

}  // namespace pwb
