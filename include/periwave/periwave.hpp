// periwave-b200: drop-in C++ API of the B200-native periodic evaluator.
//
// Same namespace, type names, field names, enumerator order and function
// signatures as the reference library's public headers
// (/root/reference/proj/include/periwave/*.hpp), so a caller of the reference
// recompiles against this header set and links libperiwave_b200.so instead.
// Everything that scales with N (near-image P2P, S2PW/PW2T contractions,
// NUFFT spreading/interpolation) runs as sm_100a CUDA kernels behind the
// C-ABI declared in include/periwave_b200.h; the types below are host-side
// descriptions (tables, options, results).
//
// Documented extensions (absent from the reference):
//   ApplyOptions::with_gradient / FieldResult::gradient (scalar kernels),
//   ApplyOptions::device / ApplyOptions::stream.
#pragma once

#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace periwave {

// ---------------------------------------------------------------- values
// (reference: include/periwave/util.hpp:12-98)
using cplx = std::complex<double>;
inline constexpr double kPi = 3.14159265358979323846264338327950288;

struct Vec2 {
  double x = 0.0, y = 0.0;
  Vec2 operator+(Vec2 o) const { return {x + o.x, y + o.y}; }
  Vec2 operator-(Vec2 o) const { return {x - o.x, y - o.y}; }
  Vec2 operator*(double s) const { return {x * s, y * s}; }
  Vec2& operator+=(Vec2 o) { x += o.x; y += o.y; return *this; }
};
inline double dot(Vec2 a, Vec2 b) { return a.x * b.x + a.y * b.y; }
inline double norm(Vec2 a) { return std::hypot(a.x, a.y); }

struct Vec2c {
  cplx x{0.0}, y{0.0};
  Vec2c operator+(const Vec2c& o) const { return {x + o.x, y + o.y}; }
  Vec2c operator-(const Vec2c& o) const { return {x - o.x, y - o.y}; }
  Vec2c& operator+=(const Vec2c& o) { x += o.x; y += o.y; return *this; }
  Vec2c operator*(cplx s) const { return {x * s, y * s}; }
};
inline Vec2c operator*(cplx s, const Vec2c& v) { return {s * v.x, s * v.y}; }

// 2x2 complex block, entries row-major (a11 a12 / a21 a22).
struct Mat2c {
  cplx a11{0.0}, a12{0.0}, a21{0.0}, a22{0.0};
  Vec2c operator*(const Vec2c& v) const { return {a11 * v.x + a12 * v.y, a21 * v.x + a22 * v.y}; }
  Mat2c operator*(cplx s) const { return {a11 * s, a12 * s, a21 * s, a22 * s}; }
  Mat2c operator+(const Mat2c& o) const { return {a11 + o.a11, a12 + o.a12, a21 + o.a21, a22 + o.a22}; }
};

// e^{-q} - 1 evaluated without cancellation near q = 0.
cplx cexpm1_neg(cplx q);

// Host fan-out helper kept for source compatibility; the product runs its
// N-scaling loops on the GPU, so this only touches host staging.
void parallel_for(std::size_t n, int nthreads, const std::function<void(std::size_t)>& fn);

// xorshift64* uniform stream, bit-identical to the reference's Rng.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  double uniform() {
    s_ ^= s_ >> 12;
    s_ ^= s_ << 25;
    s_ ^= s_ >> 27;
    return static_cast<double>((s_ * 0x2545f4914f6cdd1dull) >> 11) * 0x1.0p-53;
  }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }

 private:
  std::uint64_t s_;
};

// ---------------------------------------------------------------- errors
// (reference: include/periwave/errors.hpp:8-43; ordinal order is ABI)
enum class ErrorCode {
  NonPositiveDimension, OrientationViolation, CoincidentPoints, CoincidentSourceTarget,
  MissingBeta, InvalidOrder, OrderOutOfRange, PrecisionOutOfRange, RuleMismatch, NotDoubly,
  LengthMismatch, DimensionMismatch, NotNeutral, GridTooCoarse, OutOfInterval, NonUnitNormal,
  NotConverged, ParseError, Unsupported,
};

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void fail(ErrorCode code, const std::string& what) { throw Error(code, what); }
inline void require(bool ok, ErrorCode code, const std::string& what) {
  if (!ok) fail(code, what);
}

// ---------------------------------------------------------------- cell
// (reference: include/periwave/cell.hpp:9-68)
enum class Periodicity { Singly = 1, Doubly = 2 };

struct UnitCell {
  double d = 1.0;
  double xi = 0.0;
  double eta = 1.0;
  Periodicity periodicity = Periodicity::Doubly;
  int m0 = 1;
  Vec2 e1() const { return {d, 0.0}; }
  Vec2 e2() const { return {xi, eta}; }
};

struct LatticeTranslation {
  int m = 0, n = 0;
  Vec2 shift;
};

UnitCell make_unit_cell(double d, double xi, double eta, Periodicity periodicity);
double aspect(const UnitCell& cell);
std::vector<LatticeTranslation> near_translations(const UnitCell& cell);
Vec2 cell_coords(const UnitCell& cell, Vec2 p);
bool in_cell(const UnitCell& cell, Vec2 p);
Vec2 wrap_to_rectangle(const UnitCell& cell, Vec2 p);

struct ParticleSystem {
  std::vector<Vec2> sources;
  std::vector<double> charges;
  std::vector<Vec2> forces;
  std::vector<Vec2> normals;
  std::vector<cplx> coefficients;
  std::vector<Vec2> targets;
};

void validate_system(const UnitCell& cell, const ParticleSystem& sys);

// ---------------------------------------------------------------- kernels
// (reference: include/periwave/kernels.hpp:8-48)
enum class Pde { Poisson, ModHelmholtz, Stokes, ModStokes };

struct Mat2 {
  double a11 = 0.0, a12 = 0.0, a21 = 0.0, a22 = 0.0;
  Vec2 operator*(Vec2 v) const { return {a11 * v.x + a12 * v.y, a21 * v.x + a22 * v.y}; }
  Mat2 operator+(const Mat2& o) const { return {a11 + o.a11, a12 + o.a12, a21 + o.a21, a22 + o.a22}; }
  Mat2 operator*(double s) const { return {a11 * s, a12 * s, a21 * s, a22 * s}; }
};

double bessel_k0(double x);
double bessel_k1(double x);
double bessel_kn(int l, double x);
double greens_scalar(Pde pde, double beta, Vec2 r);
Mat2 greens_block(Pde pde, double beta, Vec2 r);
double mod_biharmonic_gmb(double beta, Vec2 r);
Vec2 pressurelet(Vec2 r);
Mat2 stresslet_dlp(Vec2 r, Vec2 n);
cplx multipole_kernel(Pde pde, double beta, int l, Vec2 r);

// ---------------------------------------------------------------- quadrature
// (reference: include/periwave/quadrature.hpp:10-66)
struct GaussRule {
  std::vector<double> nodes;
  std::vector<double> weights;
};
GaussRule gauss_legendre(int n);

struct QuadratureRule {
  std::vector<double> nodes;
  std::vector<double> weights;
  double upper = 0.0;
  int points_per_panel = 0;
  std::size_t size() const { return nodes.size(); }
};

QuadratureRule sommerfeld_rule(Pde pde, double beta, const UnitCell& cell, double eps, double min_upper = 0.0);
double certify_rule(const QuadratureRule& rule, Pde pde, double beta, const UnitCell& cell, double eps);

struct BarycentricGrid {
  double lo = 0.0;
  double hi = 0.0;
  std::vector<double> nodes;
  std::vector<double> bary_w;
  int size() const { return static_cast<int>(nodes.size()); }
};
BarycentricGrid make_barycentric_grid(double lo, double hi, int m);
std::vector<double> interp_coeffs(const BarycentricGrid& grid, double x);
int interp_nodes_for(double eps);

// ---------------------------------------------------------------- periodizer tables
// (reference: include/periwave/periodize.hpp:12-130). These are the
// plane-wave coefficient/mode tables the device plan uploads.
enum class Axis { Vertical, Horizontal };
enum class Direction { South, North, West, East };

struct ModeSet {
  Axis axis = Axis::Vertical;
  std::vector<double> phase;
  std::vector<double> decay_t;
  std::vector<double> decay_s;
  std::vector<double> shift_t;
  std::vector<double> shift_s;
  std::size_t size() const { return phase.size(); }
};

struct ScalarPart {
  Direction dir = Direction::South;
  ModeSet modes;
  std::vector<cplx> diag;
  bool take_real = true;
  bool has_m0 = false;
  double m0_coef = 0.0;
};

struct BlockPart {
  Direction dir = Direction::South;
  ModeSet modes;
  std::vector<Mat2c> diag_a;
  std::vector<Mat2c> diag_b;
  bool three_term = false;
  bool take_real = true;
  bool has_m0 = false;
  Mat2 m0_mat{0.0, 0.0, 0.0, 0.0};
};

struct PressurePart {
  Direction dir = Direction::South;
  ModeSet modes;
  std::vector<cplx> diag;
  std::vector<Vec2c> row;
  bool has_m0 = false;
  double m0_coef = 0.0;
  Vec2 m0_row{0.0, 0.0};
};

struct StressletPart {
  Direction dir = Direction::South;
  ModeSet modes;
  std::vector<Mat2c> a1, a2;
  std::vector<Mat2c> smat;
  std::vector<cplx> sa, sb;
  std::vector<cplx> off;
  bool has_m0 = false;
  double m0_coef = 0.0;
};

struct Periodizer {
  Pde pde = Pde::Poisson;
  double beta = 0.0;
  UnitCell cell;
  double eps = 1e-9;
  bool dlp = false;
  int multipole_order = 0;
  bool requires_neutrality = false;
  std::vector<ScalarPart> scalar_parts;
  std::vector<BlockPart> block_parts;
  std::vector<PressurePart> pressure_parts;
  std::vector<StressletPart> stresslet_parts;
  std::size_t rank() const;
};

int truncation_order(const UnitCell& cell, double eps);
double vertical_tail_bound(const UnitCell& cell, int M);
Periodizer make_periodizer(Pde pde, double beta, const UnitCell& cell, double eps);
Periodizer make_stokes_dlp_periodizer(const UnitCell& cell, double eps);
Periodizer make_multipole_periodizer(Pde pde, double beta, int l, const UnitCell& cell, double eps);

// ---------------------------------------------------------------- NUFFT
// (reference: include/periwave/nufft.hpp:10-31). Both backends run on the GPU.
enum class NufftBackend { Reference, Accelerated };

void nufft_type1(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& c,
                 std::size_t nmodes, std::vector<cplx>& f);
void nufft_type2(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& f,
                 std::vector<cplx>& c);
void nufft_type3(NufftBackend backend, double eps, const std::vector<double>& x, const std::vector<cplx>& c,
                 const std::vector<double>& s, std::vector<cplx>& f);
bool fast_nufft_available();

// ---------------------------------------------------------------- apply
// (reference: include/periwave/apply.hpp:13-60)
enum class ApplyPath { Auto, Direct, Accelerated };

struct ApplyOptions {
  ApplyPath path = ApplyPath::Auto;
  int threads = 1;
  bool with_pressure = false;
  double nufft_eps = 0.0;
  bool with_gradient = false;  // extension: scalar kernels, fills FieldResult::gradient
  int device = -1;             // extension: CUDA device (-1: current)
  void* stream = nullptr;      // extension: cudaStream_t to run on (nullptr: library stream)
};

struct FieldResult {
  std::vector<double> scalar;
  std::vector<Vec2> velocity;
  std::vector<double> pressure;
  std::vector<cplx> complex_scalar;
  std::vector<Vec2> gradient;  // extension
  bool accelerated = false;
};

// The documented near-field plug-in. The default accumulate runs one image
// on the GPU; total_field with no override runs all near images fused in one
// launch (bitwise not identical to per-image calls; agreement ~1e-15).
class FreeSpaceEvaluator {
 public:
  virtual ~FreeSpaceEvaluator() = default;
  virtual void accumulate(const Periodizer& pz, const ParticleSystem& sys, Vec2 shift, bool identity_shift,
                          const ApplyOptions& opt, FieldResult& out) const;
};

ApplyPath choose_path(const Periodizer& pz, std::size_t n_src, std::size_t n_tgt);
FieldResult apply_far(const Periodizer& pz, const ParticleSystem& sys, const ApplyOptions& opt = {});
FieldResult total_field(const Periodizer& pz, const ParticleSystem& sys, const ApplyOptions& opt = {},
                        const FreeSpaceEvaluator* near_eval = nullptr);

// ---------------------------------------------------------------- validation tools
// (reference: include/periwave/oracle.hpp:19-38)
FieldResult brute_force_far(const Periodizer& pz, const ParticleSystem& sys, int shells,
                            const ApplyOptions& opt = {});

struct ResidualReport {
  double e1 = 0.0;
  double e2 = 0.0;
  double scale = 0.0;
  double rel() const { return (e1 > e2 ? e1 : e2) / (scale > 1e-300 ? scale : 1e-300); }
};

ResidualReport periodicity_residual(const Periodizer& pz, const ParticleSystem& sys, int samples_per_side,
                                    const ApplyOptions& opt = {});

}  // namespace periwave
