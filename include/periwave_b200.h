/* periwave_b200.h -- C-ABI of the B200-native periodic evaluator.
 *
 * The drop-in boundary for the hot path named in BASELINE.json.north_star:
 * plain pointers, sizes and ints, no C++ or torch types, no exceptions. Every
 * entry point replaces one reference interface (file:line into
 * /root/reference/proj) and keeps its argument meaning and error behaviour:
 * an entry returns PWB_OK (0) or 1 + periwave::ErrorCode ordinal
 * (include/periwave/errors.hpp:8-28 upstream) with a thread-local message
 * from pwb_last_error(); library-side failures use the PWB_ERR_* codes >= 64.
 *
 * Memory: a pwb_system / pwb_field carries a `memory` flag. PWB_MEM_DEVICE
 * pointers are CUDA device pointers on the current device and nothing is
 * copied; PWB_MEM_HOST pointers are staged through pinned buffers by the
 * library (the end-to-end path). Positions are interleaved (x, y) doubles, the
 * same bytes as periwave::Vec2 / the reference's AoS std::vector<Vec2>, so
 * 16-byte coalesced loads need no transpose.
 *
 * Thread-safety: a pwb_periodizer is immutable after construction; its device
 * plan and scratch are per (periodizer, device) and calls on one periodizer
 * must be serialised by the caller (make one periodizer per stream for
 * concurrency). Results are run-to-run deterministic for a fixed device.
 */
#ifndef PERIWAVE_B200_H
#define PERIWAVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
enum {
  PWB_OK = 0,
  /* 1 + periwave::ErrorCode ordinal (reference include/periwave/errors.hpp:8-28) */
  PWB_ERR_NonPositiveDimension = 1,
  PWB_ERR_OrientationViolation = 2,
  PWB_ERR_CoincidentPoints = 3,
  PWB_ERR_CoincidentSourceTarget = 4,
  PWB_ERR_MissingBeta = 5,
  PWB_ERR_InvalidOrder = 6,
  PWB_ERR_OrderOutOfRange = 7,
  PWB_ERR_PrecisionOutOfRange = 8,
  PWB_ERR_RuleMismatch = 9,
  PWB_ERR_NotDoubly = 10,
  PWB_ERR_LengthMismatch = 11,
  PWB_ERR_DimensionMismatch = 12,
  PWB_ERR_NotNeutral = 13,
  PWB_ERR_GridTooCoarse = 14,
  PWB_ERR_OutOfInterval = 15,
  PWB_ERR_NonUnitNormal = 16,
  PWB_ERR_NotConverged = 17,
  PWB_ERR_ParseError = 18,
  PWB_ERR_Unsupported = 19,
  /* library-side */
  PWB_ERR_CUDA = 64,
  PWB_ERR_NO_DEVICE = 65,
  PWB_ERR_INVALID_ARGUMENT = 66,
  PWB_ERR_INTERNAL = 67
};

/* reference enums, same ordinals (kernels.hpp:17, cell.hpp:9, apply.hpp:13, nufft.hpp:19, periodize.hpp:12-13) */
enum { PWB_POISSON = 0, PWB_MODHELMHOLTZ = 1, PWB_STOKES = 2, PWB_MODSTOKES = 3 };
enum { PWB_SINGLY = 1, PWB_DOUBLY = 2 };
enum { PWB_PATH_AUTO = 0, PWB_PATH_DIRECT = 1, PWB_PATH_ACCELERATED = 2 };
enum { PWB_NUFFT_REFERENCE = 0, PWB_NUFFT_ACCELERATED = 1 };
enum { PWB_AXIS_VERTICAL = 0, PWB_AXIS_HORIZONTAL = 1 };
enum { PWB_SOUTH = 0, PWB_NORTH = 1, PWB_WEST = 2, PWB_EAST = 3 };
enum { PWB_PART_SCALAR = 0, PWB_PART_BLOCK = 1, PWB_PART_PRESSURE = 2, PWB_PART_STRESSLET = 3 };
enum { PWB_MEM_HOST = 0, PWB_MEM_DEVICE = 1 };

const char* pwb_last_error(void);
const char* pwb_version(void);
int pwb_device_count(int* count);

/* ------------------------------------------------------------ cell
 * replaces make_unit_cell (proj/src/cell.cpp:10-40 -> include/periwave/cell.hpp:41) */
typedef struct {
  double d, xi, eta;
  int periodicity; /* PWB_SINGLY | PWB_DOUBLY */
  int m0;          /* near half-width along e1, computed */
} pwb_cell;

int pwb_make_unit_cell(double d, double xi, double eta, int periodicity, pwb_cell* out);

/* near_translations (proj/src/cell.cpp:47-58): writes up to `cap` shifts
 * (x, y) and (m, n) pairs in the reference order; *count = total. */
int pwb_near_translations(const pwb_cell* cell, size_t cap, double* shifts, int* mn, size_t* count);

/* ------------------------------------------------------------ periodizer
 * replaces make_periodizer (proj/src/periodize_scalar.cpp:102-136, periodize.hpp:119),
 * make_stokes_dlp_periodizer (proj/src/periodize_stokes.cpp:302-315, periodize.hpp:122),
 * make_multipole_periodizer (proj/src/periodize_multipole.cpp:207-239, periodize.hpp:127) */
typedef struct pwb_periodizer pwb_periodizer;

int pwb_make_periodizer(int pde, double beta, const pwb_cell* cell, double eps, pwb_periodizer** out);
int pwb_make_stokes_dlp_periodizer(const pwb_cell* cell, double eps, pwb_periodizer** out);
int pwb_make_multipole_periodizer(int pde, double beta, int l, const pwb_cell* cell, double eps,
                                  pwb_periodizer** out);
void pwb_periodizer_free(pwb_periodizer* pz);
/* Periodizer::rank (proj/src/periodize_scalar.cpp:18-25) */
size_t pwb_periodizer_rank(const pwb_periodizer* pz);
/* truncation_order (proj/src/periodize_scalar.cpp:11-18) */
int pwb_truncation_order(const pwb_cell* cell, double eps, int* out);

typedef struct {
  int pde;
  double beta;
  pwb_cell cell;
  double eps;
  int dlp;
  int multipole_order;
  int requires_neutrality;
  int n_parts[4]; /* indexed by PWB_PART_* */
} pwb_periodizer_info;

int pwb_periodizer_get_info(const pwb_periodizer* pz, pwb_periodizer_info* out);

/* One part's tables (periodize.hpp:15-97). Complex values are interleaved
 * (re, im); Mat2c is 4 complex row-major (8 doubles); Vec2c is 2 complex.
 *   scalar    : t[0] diag (2/mode)                       m0[0] = m0_coef
 *   block     : t[0] diag_a (8/mode), t[1] diag_b (8)    m0[0..3] = m0_mat
 *   pressure  : t[0] diag (2), t[1] row (4)              m0 = {m0_coef, row.x, row.y}
 *   stresslet : t[0] a1, t[1] a2, t[2] smat (8 each), t[3] sa, t[4] sb, t[5] off (2 each)
 * flag = take_real (scalar, block) | three_term<<1 (block). */
typedef struct {
  int kind, axis, dir, flag, has_m0;
  size_t size;
  const double *phase, *decay_t, *decay_s, *shift_t, *shift_s;
  const double* t[6];
  double m0[4];
} pwb_part;

/* Views into the periodizer's host tables; valid until pwb_periodizer_free. */
int pwb_periodizer_get_part(const pwb_periodizer* pz, int kind, int index, pwb_part* out);
/* Build a periodizer from externally supplied tables (e.g. parts exported by
 * another builder); the tables are copied. */
int pwb_periodizer_new(int pde, double beta, const pwb_cell* cell, double eps, int dlp, int multipole_order,
                       int requires_neutrality, pwb_periodizer** out);
int pwb_periodizer_add_part(pwb_periodizer* pz, const pwb_part* part);

/* ------------------------------------------------------------ particles, options, results */
typedef struct {
  size_t n_src, n_tgt;
  const double* sources;      /* 2*n_src */
  const double* charges;      /* n_src or NULL   (ParticleSystem::charges) */
  const double* forces;       /* 2*n_src or NULL (ParticleSystem::forces) */
  const double* normals;      /* 2*n_src or NULL (ParticleSystem::normals) */
  const double* coefficients; /* 2*n_src or NULL (ParticleSystem::coefficients, re/im) */
  const double* targets;      /* 2*n_tgt */
  int memory;                 /* PWB_MEM_HOST | PWB_MEM_DEVICE */
} pwb_system;

typedef struct {
  int path;          /* ApplyOptions::path */
  int threads;       /* ApplyOptions::threads (host staging only) */
  int with_pressure; /* ApplyOptions::with_pressure */
  double nufft_eps;  /* ApplyOptions::nufft_eps (0: derived) */
  int with_gradient; /* extension (scalar kernels): fill pwb_field::gradient */
  int device;        /* CUDA device, -1 = current */
  void* stream;      /* cudaStream_t, NULL = the library's per-periodizer stream (a blocking
                        stream: ordered after legacy-default-stream work) */
} pwb_options;

void pwb_options_default(pwb_options* opt);

typedef struct {
  double* scalar;         /* n_tgt   FieldResult::scalar */
  double* velocity;       /* 2*n_tgt FieldResult::velocity */
  double* pressure;       /* n_tgt   FieldResult::pressure */
  double* complex_scalar; /* 2*n_tgt FieldResult::complex_scalar */
  double* gradient;       /* 2*n_tgt extension */
  int accelerated;        /* out: FieldResult::accelerated */
  int memory;             /* PWB_MEM_HOST | PWB_MEM_DEVICE */
} pwb_field;

/* ------------------------------------------------------------ apply (the hot path)
 * total_field (proj/src/apply.cpp:548-556, apply.hpp:58-60): far apply plus the
 *   fused near images; the output arrays of the periodizer's kind are overwritten.
 * apply_far (proj/src/apply.cpp:417-479, apply.hpp:52-53): overwritten.
 * accumulate = FreeSpaceEvaluator::accumulate (proj/src/apply.cpp:481-546,
 *   apply.hpp:42-44): ADDS one image's direct sum into *out.
 * near_field: ADDS every near_translations image (one fused launch).
 * Host systems (PWB_MEM_HOST) whose targets hold the same bytes as their sources are staged
 * as one device array (the symmetric near tile). Small total_field calls (one-sided near
 * tile, N_S N_T <= ~4.2e6) replay a CUDA graph captured on their second repetition with the
 * same pointers and sizes (PWB_NO_GRAPH=1 disables it); errors are still returned, but the
 * device output arrays of such a failed call are unspecified. */
int pwb_total_field(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out);
int pwb_apply_far(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out);
int pwb_accumulate(const pwb_periodizer* pz, const pwb_system* sys, double shift_x, double shift_y,
                   int identity_shift, const pwb_options* opt, pwb_field* out);
int pwb_near_field(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out);
/* choose_path (proj/src/apply.cpp:409-415, apply.hpp:48) */
int pwb_choose_path(const pwb_periodizer* pz, size_t n_src, size_t n_tgt, int* path);

/* Sharded far field (multi-GPU). The coefficient buffer is
 * linear in the sources: each rank runs the source pass on its source slice,
 * the caller sums the buffers (ncclAllReduce, fp64, sum), then every rank runs
 * the target pass on its target slice. Buffer = `*n_doubles` device doubles. */
int pwb_far_coeff_size(const pwb_periodizer* pz, const pwb_options* opt, size_t n_src_total, size_t n_tgt_total,
                       size_t* n_doubles);
int pwb_far_source_pass(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt,
                        size_t n_src_total, size_t n_tgt_total, double* coeff_dev);
int pwb_far_target_pass(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt,
                        size_t n_src_total, size_t n_tgt_total, const double* coeff_dev, pwb_field* out);
/* Sharded symmetric near field (targets == sources). The unordered pairs are cut
 * into `*n_items` work items (host-only query); each rank runs a disjoint item
 * range into its own fixed-point accumulator acc (device, zeroed by the caller,
 * n * nout * 3 int64, target-major: acc[(l*nout + c)*3 + limb]); the accumulators
 * are summed exactly as integers (e.g. ncclReduceScatter(ncclInt64, sum) so each
 * rank receives a contiguous slice of targets), and pwb_fixed_to_field adds a
 * slice into the outputs. Bitwise deterministic for any split.
 * The accumulator holds the near field times 2^scale_exp (*scale_exp, written by
 * pwb_near_sym_partial; derived from max |strength| and n, hence identical on every rank
 * that holds the same strengths): pass it to pwb_fixed_to_field.
 * *status: bit 0 = a non-identity exact coincidence (the reference's
 * CoincidentSourceTarget, apply.cpp:544-545), bit 1 = the fixed-point range was exceeded
 * (non-finite strengths). The call does NOT raise these (returns PWB_OK), so that every
 * rank can combine the status words (e.g. allreduce MAX) before the reduce-scatter and
 * raise the same error everywhere instead of leaving peers blocked in a collective. */
int pwb_near_sym_items(const pwb_periodizer* pz, size_t n, const pwb_options* opt, long* n_items, int* nout);
int pwb_near_sym_partial(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, long item_begin,
                         long item_end, int64_t* acc, int* scale_exp, int* status);
/* Item boundaries bounds[0..world] (host array of world + 1, world <= 64) of a balanced split of
 * the symmetric work items over `world` ranks: rank r runs [bounds[r], bounds[r+1]). For the
 * screened kernels (modified Helmholtz) the split balances the estimated cost per item from
 * the tile bounding boxes (their image masks and regimes make item costs differ); for the
 * others it is the even split by count. Same inputs give the same bounds on every rank.
 * Extension (multi-GPU; no reference counterpart). */
int pwb_near_sym_split(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, int world,
                       long* bounds);
int pwb_fixed_to_field(const pwb_periodizer* pz, const pwb_options* opt, const int64_t* acc, size_t n_targets,
                       int scale_exp, pwb_field* out);
/* Strength/neutrality/cell checks of apply_far (proj/src/apply.cpp:350-393, cell.cpp:77-94),
 * evaluated on the device for device-resident systems. */
int pwb_validate(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt);

/* ------------------------------------------------------------ validation tools (GPU)
 * brute_force_far (proj/src/oracle.cpp:83-110, oracle.hpp:30-31): shell-by-shell
 *   +-paired lattice sum of the images outside the near set (each image one GPU
 *   accumulate launch), early stop after 3 quiet shells; overwrites *out. Host memory.
 * periodicity_residual (proj/src/oracle.cpp:112-173, oracle.hpp:43-44): face jumps of
 *   total_field over samples_per_side points per face; the system's targets are ignored. */
int pwb_brute_force_far(const pwb_periodizer* pz, const pwb_system* sys, int shells, const pwb_options* opt,
                        pwb_field* out);
int pwb_periodicity_residual(const pwb_periodizer* pz, const pwb_system* sys, int samples_per_side,
                             const pwb_options* opt, double* e1, double* e2, double* scale);

/* ------------------------------------------------------------ NUFFT
 * nufft_type1/2/3 (proj/src/nufft.cpp:71-82, nufft.hpp:21-31). Complex arrays
 * interleaved; `memory` applies to every array argument. */
int pwb_nufft_type1(int backend, double eps, size_t n, const double* x, const double* c, size_t nmodes, double* f,
                    int memory, void* stream);
int pwb_nufft_type2(int backend, double eps, size_t n, const double* x, size_t nmodes, const double* f, double* c,
                    int memory, void* stream);
int pwb_nufft_type3(int backend, double eps, size_t n, const double* x, const double* c, size_t nk, const double* s,
                    double* f, int memory, void* stream);
/* fast_nufft_available (proj/src/nufft_fast.cpp:211) */
int pwb_fast_nufft_available(void);

/* ------------------------------------------------------------ pair kernels on the device
 * Batch evaluation of the device functions the P2P tiles use (kernels.cpp:78-162),
 * for parity tests. which: 0 bessel_kn(l, x); 1 greens_scalar(pde, beta, r);
 * 2 greens_block (4 out); 3 multipole_kernel(pde, beta, l, r) (2 out);
 * 4 pressurelet (2 out); 5 stresslet_dlp(r, n) (4 out); 6 the symmetric tiles'
 * ln(x) in both precision tiers, the MUFU reciprocal seed, the refined 1/x,
 * the MUFU reciprocal-square-root seed and the refined 1/sqrt(x) (6 out, no
 * reference counterpart); 7 the near tiles' K0(x), K1(x)
 * in the full and the reduced tier (4 out, x < 64); 8 the reduced tier's table-driven
 * ln(x) (1 out); 9 K0(x), K1(x) in the symmetric screened tile's coarse tier (2 out,
 * x < 64); 10 the coarse table-driven ln(x) (1 out); 11 the reciprocal-seeded coarse ln(x)
 * of the product-form Laplace tile (1 out); 12 the hardware reciprocal seed of x's high
 * word with its low 12 bits cleared (1 out). Inputs per point: which 0, 6-12: x (1 double);
 * 1-4: r (2); 5: r, n (4).
 * Host memory. */
int pwb_eval_kernel(int which, int pde, double beta, int l, size_t n, const double* in, double* out);

/* ------------------------------------------------------------ measurement */
/* Kernels launched by this process through the engine (bench gpu_launches). */
int pwb_launch_count(long* count);
/* Device time of the last apply on this periodizer/device: far (S2PW + PW2T)
 * and near (the fused P2P tile launch), from CUDA events on the launch stream. */
int pwb_last_phase_ms(const pwb_periodizer* pz, int device, double* far_ms, double* near_ms);
/* Best-of DFMA-chain throughput of the device in TFLOP/s (roofline denominator;
 * MEASURED_PEAKS.json has no fp64 entry). */
int pwb_fp64_peak_probe(int device, double* tflops);

/* ------------------------------------------------------------ utilities */
/* Rng::uniform stream (proj/include/periwave/util.hpp:83-98), host memory. */
int pwb_rng_uniform(uint64_t seed, size_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PERIWAVE_B200_H */
