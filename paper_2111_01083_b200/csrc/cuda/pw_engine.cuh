// Internal device-engine interface shared by the kernel translation units and
// the host orchestration (engine.cu). Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

namespace pwb {

constexpr int kMaxImg = 21;   // doubly periodic m0 <= 3: 7 x 3 images
constexpr int kMaxSplits = 64;

struct CudaFailure : std::runtime_error {
  explicit CudaFailure(const std::string& s) : std::runtime_error(s) {}
};
struct InternalFailure : std::runtime_error {
  explicit InternalFailure(const std::string& s) : std::runtime_error(s) {}
};
[[noreturn]] void throw_internal(const char* what);
void cuda_check(cudaError_t e, const char* what);
// Number of kernels this process has launched through the engine (pwb_launch_count).
void count_launches(long n);
long launch_count();
// Max shared-memory carveout for a kernel, once per (device, kernel).
void set_max_carveout(const void* kernel);

// ---------------------------------------------------------------- fixed-point scale
// Exponent k of the symmetric tile's fixed-point scale 2^k (near_sym_impl.cuh fx_add):
// maxhi = high word of max |strength| (its bit order is the order of the non-negative
// doubles), n = number of sources; 2^e > max |strength| and 2^lg >= n, so the scaled
// sum of |strength| over all sources is below 2^24. Non-finite or all-zero strengths: 0.
__host__ __device__ inline int fx_exponent(unsigned maxhi, size_t n) {
  if (maxhi == 0u || maxhi >= 0x7ff00000u) return 0;
  const int e = static_cast<int>(maxhi >> 20) - 1023 + 1;
#ifdef __CUDA_ARCH__
  const int lg = n > 1 ? 64 - __clzll(static_cast<long long>(n - 1)) : 0;
#else
  const int lg = n > 1 ? 64 - __builtin_clzll(static_cast<unsigned long long>(n - 1)) : 0;
#endif
  const int k = 24 - e - lg;
  return k < -960 ? -960 : (k > 960 ? 960 : k);
}
__host__ __device__ inline double fx_scale(int k) {  // 2^k, |k| <= 960
  const long long bits = static_cast<long long>(1023 + k) << 52;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(bits);
#else
  double v;
  std::memcpy(&v, &bits, sizeof v);
  return v;
#endif
}

// ---------------------------------------------------------------- near field
enum class NearKind { Laplace, ModHelm, ModHelmGrad, Stokes, StokesP, ModStokes, ModStokesP, Stresslet, Multipole };

struct NearArgs {
  const double2* tgt = nullptr;
  size_t nt = 0;
  const double2* src = nullptr;
  size_t ns = 0;
  const double* q = nullptr;       // charges
  const double2* vec = nullptr;    // forces or complex coefficients
  const double2* nrm = nullptr;    // normals (stresslet)
  double shx[kMaxImg] = {};        // row-major [n][m]: m*d + n*xi (reference association)
  double shy[3] = {};              // n*eta
  int nxi = 1, nrow = 1, id_img = -1;
  double beta = 0.0, beta2 = 0.0, xcut2 = 0.0, ms_scale = 0.0;
  int order = 0, screened = 0;
  double* out0 = nullptr;  // first nout0 outputs, interleaved per target
  int nout0 = 1;
  double* out1 = nullptr;  // remaining outputs (gradient / pressure)
  int nout1 = 0;
  double* partial = nullptr;
  int splits = 1;
  size_t src_per_split = 0;
  int* flag = nullptr;     // bit 0: a non-identity exact coincidence; bit 1: fixed-point range exceeded
  const unsigned* fx_maxhi = nullptr;  // symmetric tiles: high word of max |strength| (launch_fx_maxhi)
  const int* out_row = nullptr;  // binned targets: output row of target l (nullptr: l)
  int lowp = 0;                  // near tiles: reduced-precision tier (eps >= 1e-11, pw_math.cuh)
  int cull = 1;                  // screened symmetric tiles: per-tile image mask (near_sym_impl.cuh)
  int unskewed = 0;              // fused layout with shx[n][m] independent of n (xi == 0)
  int coarse_log = 0;            // symmetric Laplace / Stokeslet tiles: 256-entry table log (eps >= 1e-10)
  double cheb_tol = 0.0;         // screened symmetric tile: per-tile-pair Chebyshev K0 fit (0: off)
  double inv_beta2 = 0.0;
  // Product-form symmetric tiles (near_sym_impl.cuh SymLaplace / SymStokes PROD):
  // src / tgt hold the binned points times prod_sc: 2 / d when that is an exact power of two,
  // so the period is 2 in the tile's units, else 1 (0: off)
  double prod_sc = 0.0;
  double prod_log_off = 0.0;     // ln(16 / prod_sc^6) (Laplace), ln(512 / prod_sc^18) (Stokeslet): added to the log table's entries
  double prod_ln_sc2 = 0.0;      // ln(prod_sc^2): one image's log offset on the careful path
  double prod_eta = 0.0;         // eta * prod_sc: the image rows' offset in the tile's units (3 x 3 images)
  int prod = 0;                  // 0: off; 1: points scaled to period 2; 2: unscaled points (prod_sc = 1), any period
  double prod_period = 2.0;      // the period in the tile's units: 2 (scaled) or d
  double prod_d2 = 0.0, prod_4d2 = 0.0;  // unscaled form: d^2, 4 d^2
  // host side only: a split one-sided tile may run on its own stream (a parallel branch of a
  // captured small call, engine.cu total_eager); the partials' reduction waits for tile_done
  void* tile_stream = nullptr;
  void* tile_done = nullptr;
};

// ---------------------------------------------------------------- spatial binning (binning.cu)
struct BinBox {  // uniform grid: cell = floor((p - (x0, y0)) * inv_h), 16 bits per axis
  double x0 = 0.0, y0 = 0.0, inv_h = 1.0;
};
size_t morton_order_bytes(size_t n);
// perm[i] = index of the i-th point in Morton order (stable in the input index).
void morton_order(const double2* pts, size_t n, const BinBox& box, int* perm, void* ws, size_t ws_bytes,
                  cudaStream_t st);
void gather_double(const double* in, const int* perm, size_t n, double* out, cudaStream_t st);
void gather_double2(const double2* in, const int* perm, size_t n, double2* out, cudaStream_t st);
// out[i] = in[perm[i]] * sc (sc a power of two: exact)
void gather_scale_double2(const double2* in, const int* perm, size_t n, double sc, double2* out, cudaStream_t st);
// out[perm[i]] += in[i] row-wise (width uint64 per row): sorted fixed-point rows -> input order
void scatter_add_rows(const unsigned long long* in, const int* perm, size_t n, int width, unsigned long long* out,
                      cudaStream_t st);

size_t near_outputs(NearKind kind);
void launch_near(NearKind kind, const NearArgs& a, cudaStream_t st, double* partial_ws, int sm_count);
// Symmetric (targets == sources) fused near images: each unordered pair once
// (near_sym.cu). fx: 3 * n * nout uint64 accumulators; row_start: nb + 1 int64
// (device and pinned host). Returns false when the kind/layout has no symmetric form.
bool near_sym_supported(NearKind kind);
size_t near_sym_tiles(size_t n);
// Work-item range of one launch: the default is the whole triangle with the
// accumulator zeroed first and converted into the outputs at the end (finish);
// multi-GPU ranks run disjoint item ranges into their own accumulator (finish =
// false), sum the accumulators (integer reduce-scatter) and convert their slice.
struct SymRange {
  long begin = -1, end = -1;
  bool finish = true;
  bool count_only = false;
  long* total_items = nullptr;
};
bool launch_near_sym(NearKind kind, const NearArgs& a, cudaStream_t st, unsigned long long* fx,
                     long long* row_start_dev, long long* row_start_host, const SymRange& range);
// *maxhi = high word of max over the sources of |q| / |f.x|, |f.y| (zeroed first).
void launch_fx_maxhi(const NearArgs& a, unsigned* maxhi, cudaStream_t st);
// out += fixed-point accumulators * 2^-k, k = fx_exponent(*maxhi_dev, n_src) when maxhi_dev
// is given, else k_host; skipped entirely when flag bit 1 (overflow) is set.
void launch_fx_finish(const unsigned long long* fx, size_t n, double* out0, int nout0, double* out1, int nout1,
                      const int* out_row, const unsigned* maxhi_dev, size_t n_src, int k_host, const int* flag,
                      cudaStream_t st);
// host-only: number of work items of the symmetric decomposition (0 if none)
// (prod: a product-form tile runs, NearArgs::prod != 0)
long near_sym_item_count(NearKind kind, size_t n, bool prod = false);
// Tile size (points) and column tiles per work item of the symmetric tile of `kind`.
void near_sym_shape(NearKind kind, int* tile, int* chunk);
// Cost-balanced item boundaries (world + 1 longs, host) for the screened symmetric tiles:
// tile boxes of the (binned) points in a.tgt, estimated item costs, prefix sum, split.
size_t near_sym_split_bytes(size_t n, long items);
void near_sym_split(NearKind kind, const NearArgs& a, int world, long* bounds_host, void* ws, size_t ws_bytes,
                    long long* row_start_dev, long long* row_start_host, cudaStream_t st);

// ---------------------------------------------------------------- far field (direct S2PW / PW2T)
// Weight sets: what each source contributes per mode (K real weights).
enum class WeightSet { Charge = 1, Coef = 2, Force = 3, ForceW = 4, DoubleLayer = 5 };

inline int weight_count(WeightSet w) {
  switch (w) {
    case WeightSet::Charge: return 1;
    case WeightSet::Coef:
    case WeightSet::Force: return 2;
    case WeightSet::ForceW: return 4;
    case WeightSet::DoubleLayer: return 8;
  }
  return 1;
}

struct ModeTable {  // device SoA, one entry per mode of a family
  const double* phase = nullptr;
  const double* decay_t = nullptr;
  const double* decay_s = nullptr;
  const double* shift_t = nullptr;
  const double* shift_s = nullptr;
  const int* axis = nullptr;  // 0 vertical (w = y, p = x), 1 horizontal (w = x, p = y)
  int count = 0;
};

struct S2pwArgs {
  ModeTable modes;
  const double2* src = nullptr;
  const double* q = nullptr;
  const double2* vec = nullptr;
  const double2* nrm = nullptr;
  size_t ns = 0;
  size_t per_chunk = 0;
  int chunks = 1;
  double* partial = nullptr;  // [chunk][mode][K][2] (chunks == 1: the raw sums themselves)
  int narrow = 0;             // 1: one mode per block (small problems: more blocks, shorter chains)
};
// small source counts take one chunk and one mode per block (s2pw_kernel<WS, 1>)
constexpr size_t kS2pwNarrowSources = 4096;
void launch_s2pw(WeightSet ws, const S2pwArgs& a, cudaStream_t st);
// sums partial over chunks (fixed order) into raw[mode][K][2]
void launch_chunk_sum(const double* partial, int chunks, size_t per_chunk_len, double* raw, cudaStream_t st);

// target side: acc += T_l(r) (A_r + w_l B_r), KO complex outputs per target
struct Pw2tArgs {
  ModeTable modes;
  const double* A = nullptr;  // [mode][KO][2]
  const double* B = nullptr;  // [mode][KO][2] or nullptr
  const double2* tgt = nullptr;
  size_t nt = 0;
  int ko = 1;
  int gradient = 0;             // scalar family only: also d/dx, d/dy
  const double* m0_lin = nullptr;    // [KO][2] device, acc += y * m0_lin (nullable)
  const double* m0_const = nullptr;  // [KO][2] device, acc += m0_const (nullable)
  // outputs: Re of each complex component, or complex pairs
  double* out_re = nullptr;     // real output, KO per target (overwrite or add)
  double* out_cplx = nullptr;   // complex output, KO complex per target
  double* out_grad = nullptr;   // gradient (2 per target)
  int accumulate = 0;           // add into outputs instead of overwriting
};
void launch_pw2t(const Pw2tArgs& a, cudaStream_t st);

// per-mode finalisation of the raw source sums into target coefficients A/B
enum class FamilyKind { Scalar = 0, Block = 1, Pressure = 2, Stresslet = 3 };
struct PrepArgs {
  FamilyKind kind = FamilyKind::Scalar;
  int count = 0;
  int k = 1;            // weights per source
  const double* raw = nullptr;   // [mode][K][2]
  const double* t0 = nullptr;    // family tables (see engine.cu)
  const double* t1 = nullptr;
  const double* t2 = nullptr;
  const double* t3 = nullptr;
  const double* t4 = nullptr;
  const double* t5 = nullptr;
  const int* three_term = nullptr;  // block: per mode flag
  double* A = nullptr;
  double* B = nullptr;
};
void launch_prep(const PrepArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- reductions / validation
// moments over sources: [sum y q, sum y fx, sum y fy, sum n2 fx + n1 fy, sum n1 fx + n2 fy]
constexpr int kMoments = 5;
// validation: [bad points, bad normals, sum q, sum |q|, sum fx, sum fy, sum |f|, sum re c, sum im c, sum |c|]
constexpr int kChecks = 10;
struct ReduceArgs {
  const double2* src = nullptr;
  const double* q = nullptr;
  const double2* vec = nullptr;  // forces
  const double2* coef = nullptr;
  const double2* nrm = nullptr;
  size_t ns = 0;
  const double2* tgt = nullptr;
  size_t nt = 0;
  double d = 1.0, xi = 0.0, eta = 1.0;
};
constexpr int kReduceBlocks = 296;
// blocks of the validation / moment reduction for n points: 296 (2 per SM) from ~76K points
// on, one per 256 points below (c1: 4), so the block partials' final sum stays short
inline int reduce_blocks(size_t n) {
  const size_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > static_cast<size_t>(kReduceBlocks) ? kReduceBlocks : b));
}
// writes per-block partials: moments [blocks][kMoments], checks [blocks][kChecks]
void launch_reduce(const ReduceArgs& a, double* block_moments, double* block_checks, int blocks, cudaStream_t st);
void launch_sum_blocks(const double* block_vals, int blocks, int n, double* out, cudaStream_t st);

// ---------------------------------------------------------------- NUFFT lines (nufft.cu)
constexpr int kMaxLines = 64;

// Legendre interpolation grid (quadrature.cpp:258-304) in reference coordinates.
struct BaryGrid {
  double lo = 0.0, hi = 0.0;
  int m = 0;  // 0: no barycentric lines (a single line of weight 1)
  double tk[kMaxLines] = {};
  double bw[kMaxLines] = {};
};

enum class PosKind : int { Array = 0, WrappedX = 1, PointY = 2 };

struct SpreadArgs {
  size_t n = 0;                  // points
  PosKind pos = PosKind::Array;  // how the spreading coordinate is formed
  const double* xs = nullptr;    // PosKind::Array
  const double2* pts = nullptr;  // WrappedX / PointY (also the barycentric coordinate source)
  double d = 1.0, kx = 1.0;      // WrappedX: -wrap(x, d) * kx
  const double* c = nullptr;     // strengths (spread only)
  int cplx = 0;                  // strengths complex interleaved (else real)
  int open = 0;                  // open grid (type 3): t = p / hx + nf / 2
  double h = 1.0, inv_h = 1.0;
  int nf = 0, w = 3;
  double beta = 6.9;
  int lines = 1, lpg = 1;
  BaryGrid bary;                 // line weights from the barycentric row (m > 0)
  int bary_axis = 0;             // 0: y coordinate, 1: x coordinate of pts
  size_t per_chunk = 0;
};

struct MixArgs {
  int nmodes = 0, lines = 0;
  const int* bucket_start = nullptr;  // [nmodes + 1]
  const int* bucket = nullptr;        // mode ids (vertical family indices), part order
  const double *decay_s = nullptr, *shift_s = nullptr, *decay_t = nullptr, *shift_t = nullptr;
  const double* diag = nullptr;       // complex per mode
  const double* nodes = nullptr;      // [lines] interpolation nodes (device)
};

}  // namespace pwb
