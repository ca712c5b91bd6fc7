// Device plan and orchestration of one apply (host side of the engine).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "periwave/periwave.hpp"
#include "pw_engine.cuh"

namespace pwb {

// cuFFT plans of one owner (a device Plan, or one standalone transform call), keyed by
// (nf, lines): every owner has its own handles and work areas, made on the owner's
// device, so two Plans (two devices, or two streams in two threads) never share a work
// area; the handles are destroyed with their owner (nufft.cu).
class FftPlans {
 public:
  FftPlans() = default;
  FftPlans(const FftPlans&) = delete;
  FftPlans& operator=(const FftPlans&) = delete;
  ~FftPlans();
  // batched in-place complex transform of `lines` lines of nf points; sign +1 = e^{+i}
  void exec(double* data, int nf, int lines, int sign, cudaStream_t st);

 private:
  std::map<std::pair<int, int>, int> plans_;  // cufftHandle is an int
};

// Bumped whenever a DevBuf / PinnedBuf moves (grows): captured CUDA graphs hold raw
// workspace pointers and are dropped when it changes (Plan::total_graphed).
unsigned long buffer_epoch();

// RAII device buffer that only grows.
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void* ensure(size_t bytes);
  template <class T>
  T* as(size_t count) {
    return static_cast<T*>(ensure(count * sizeof(T)));
  }
  void* get() const { return p_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

class PinnedBuf {
 public:
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf();
  void* ensure(size_t bytes);

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

// Device view of a particle system (positions interleaved like periwave::Vec2).
struct DevSys {
  const double2* src = nullptr;
  const double* q = nullptr;
  const double2* f = nullptr;
  const double2* nrm = nullptr;
  const double2* coef = nullptr;
  size_t ns = 0;
  const double2* tgt = nullptr;
  size_t nt = 0;
};

struct DevOut {
  double* scalar = nullptr;
  double* velocity = nullptr;
  double* pressure = nullptr;
  double* complex_scalar = nullptr;
  double* gradient = nullptr;
};

struct Opts {
  periwave::ApplyPath path = periwave::ApplyPath::Auto;
  bool with_pressure = false;
  bool with_gradient = false;
  double nufft_eps = 0.0;
  cudaStream_t stream = nullptr;
};

enum class Kind { Scalar, Velocity, Multipole };
Kind kind_of(const periwave::Periodizer& pz);
// which near-field tile the periodizer and options select (host only)
NearKind near_kind_of(const periwave::Periodizer& pz, bool with_pressure, bool with_gradient);
// whether the symmetric near field of n points takes the product-form Laplace tile (host-only)
bool prod_eligible(const periwave::Periodizer& pz, NearKind nk, size_t n);

// One family of plane-wave parts that share a weight set and output shape.
struct Family {
  FamilyKind kind = FamilyKind::Scalar;
  WeightSet ws = WeightSet::Charge;
  int count = 0;
  int ko = 1;
  bool pressure = false;  // only when ApplyOptions::with_pressure
  DevBuf phase, decay_t, decay_s, shift_t, shift_s, axis;
  DevBuf t[6];
  DevBuf three_term;
  // rank-one terms: out += (y * lin + cst) with lin/cst = M * (moment[ia], moment[ib])
  bool has_lin = false, has_cst = false;
  int ia = 0, ib = 0;
  double mlin[4] = {0, 0, 0, 0};
  double mcst[2] = {0, 0};
  size_t raw_offset = 0;  // in the coefficient buffer (doubles)
  int axis_group = 0;     // scalar families: 0 vertical parts, 1 horizontal parts
  std::vector<double> host_phase;
  std::vector<int> part_sizes;  // modes per part, in part order
  ModeTable table() const;
};

// Accelerated vertical route (apply.cpp:200-259): Legendre lines in y, one type-1
// transform per line on the sources, mode mixing, one type-2 per line on the targets.
struct VertAccel {
  bool ready = false;
  int mmax = 0, nmodes = 0, mg = 0;
  double lo = 0.0, hi = 0.0;
  std::vector<double> nodes_host;
  DevBuf nodes, bucket_start, bucket;
  // per inner eps
  double eps = -1.0;
  int nf = 0, w = 0;
  double beta = 0.0;
  DevBuf fac;
  // BaryGrid is filled at build time (device copies live in the kernel parameters)
  double tk[64] = {}, bw[64] = {};
};

// Accelerated horizontal route of singly periodic cells (apply.cpp:261-348): Legendre
// lines in x, per part one type-3 transform per line on the sources (y -> -lambda)
// and one on the targets (lambda -> y). The interval and the y extents are the
// closed cell's (data-independent, so every rank of a sharded apply builds the
// same grids).
struct HorizAccel {
  bool ready = false;
  int mg = 0;
  double lo = 0.0, hi = 0.0, ymax = 0.0, lmax = 0.0;
  double tk[64] = {}, bw[64] = {};
  DevBuf nodes, neg_lam;
  std::vector<int> part_start;  // mode ranges of the parts inside the horizontal family
  // per inner eps
  double eps = -1.0;
  int w = 0, nf1 = 0, nf2 = 0, ngl = 0;
  double beta = 0.0, hx1 = 0.0, hx2 = 0.0;
  DevBuf fac1, gl_amp, gl_z;
};

class Plan {
 public:
  Plan(const periwave::Periodizer& pz, int device);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  int device() const { return device_; }
  cudaStream_t stream_for(const Opts& o) const { return o.stream ? o.stream : stream_; }

  // apply_far's checks (apply.cpp:417-422, :350-393) on a device-resident system
  void validate(const DevSys& s, const Opts& o, bool far_checks, bool neutrality = true);
  // the path Auto resolves to for the whole (possibly sharded) problem (apply.cpp:424)
  periwave::ApplyPath resolve(const Opts& o, size_t n_src_total, size_t n_tgt_total) const;
  size_t coeff_size(const Opts& o, periwave::ApplyPath path);
  // moments_ready: validate(far_checks) of the same system just ran (its block moments are reused)
  // moments_after: an event (the validation branch of a captured call) the moment sum waits for
  void source_pass(const DevSys& s, const Opts& o, double* coeff, periwave::ApplyPath path,
                   bool moments_ready = false, cudaEvent_t moments_after = nullptr);
  // returns the accelerated flag (apply.cpp:464-471)
  bool target_pass(const DevSys& s, const Opts& o, const double* coeff, const DevOut& out, periwave::ApplyPath path);
  // adds every near image (fused) or one image (single shift)
  void near(const DevSys& s, const Opts& o, const DevOut& out, bool single, double shx, double shy, bool identity);
  // multi-GPU symmetric near field: work items of the triangle decomposition for n
  // points, a range of them into a fixed-point accumulator, and its conversion
  long sym_items(const Opts& o, size_t n);
  int near_nout(const Opts& o) const;
  // returns status bits (1: coincidence, 2: fixed-point range exceeded) instead of throwing,
  // so every rank can agree on the error before a collective; *scale_exp = the exponent k
  // of the fixed-point scale (fx_exponent) the accumulator is in
  int sym_partial(const DevSys& s, const Opts& o, long begin, long end, unsigned long long* acc, int* scale_exp);
  // item boundaries [world + 1] of a balanced multi-GPU split of the symmetric items
  void sym_split(const DevSys& s, const Opts& o, int world, long* bounds);
  void fixed_finish(const Opts& o, const unsigned long long* acc, size_t n, int scale_exp, const DevOut& out);
  // full pipeline on device pointers; returns the accelerated flag. Small one-sided
  // problems replay a captured CUDA graph of the whole sequence (validation reductions,
  // far passes, near tile, status copies) with one host synchronisation.
  bool total(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images);

  std::mutex& mutex() { return mu_; }
  // device time (ms) of the last call's phases: [validate+far, near]
  void phase_ms(double* far_ms, double* near_ms);

  // staging for host-memory calls
  DevBuf stage[8];
  PinnedBuf pin;

 private:
  // declared first, destroyed last: ~Plan makes the plan's device current for the member
  // destructors (cuFFT handles, device buffers) and this restores the caller's device
  struct RestoreDevice {
    int prev = -1;
    ~RestoreDevice() {
      if (prev >= 0) cudaSetDevice(prev);
    }
  } restore_;
  const periwave::Periodizer& pz_;
  int device_ = 0;
  int sms_ = 148;
  cudaStream_t stream_ = nullptr;
  std::vector<std::unique_ptr<Family>> fams_;
  DevBuf s2pw_partial_, coeff_ws_, A_, B_, m0_, near_partial_, flag_, red_m_, red_c_, red_out_;
  PinnedBuf host_checks_;
  int moment_blocks_ = kReduceBlocks;  // blocks of the last validation reduce (its partials in red_m_)
  DevBuf sym_fx_, sym_rows_, sym_split_ws_, fx_maxhi_;
  PinnedBuf sym_rows_host_;
  // spatially binned copies of the near-field inputs (binning.cu)
  DevBuf bin_ws_, bin_perm_s_, bin_perm_t_, bin_src_, bin_tgt_, bin_q_, bin_vec_, bin_nrm_;
  void bin_inputs(const DevSys& s, NearArgs& a, cudaStream_t st);
  std::mutex mu_;
  cudaEvent_t ev_[4] = {nullptr, nullptr, nullptr, nullptr};
  bool far_timed_ = false, near_timed_ = false;

  // ---- CUDA-graph replay of small calls (launch-latency bound: c1 is 15 launches of a
  // few microseconds each). A call shape (every pointer, size and option) seen twice is
  // captured once; the validation and coincidence checks are deferred to after the
  // single synchronisation (the call still raises; outputs are unspecified on error).
  struct GraphKey {
    DevSys s;
    unsigned outs = 0;  // which outputs are requested (bit i: scalar, velocity, pressure, complex, gradient)
    int path = 0;
    bool pressure = false, gradient = false, far = false, near = false;
    double nufft_eps = 0.0;
    bool operator==(const GraphKey& o) const;
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    long launches = 0;
    bool accelerated = false, far_timed = false, near_timed = false;
    std::vector<std::function<void()>> checks;
  };
  bool graph_eligible(const DevSys& s, bool far, bool near_images) const;
  bool total_eager(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images);
  bool total_graphed(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images);
  void drop_graphs();
  void record(int i, cudaStream_t st);
  bool defer_ = false;                          // checks go to pending_ instead of syncing
  std::vector<std::function<void()>> pending_;  // deferred checks of the call being captured
  std::vector<GraphEntry> graphs_;
  std::vector<GraphKey> seen_;
  std::vector<GraphKey> no_graph_;  // shapes whose capture failed: eager from then on
  unsigned long graph_epoch_ = 0;
  cudaStream_t capture_stream_ = nullptr;
  // parallel branches of a captured call: [0] validation, [1] the near tile
  cudaStream_t side_[2] = {nullptr, nullptr};
  cudaEvent_t fork_ev_ = nullptr, side_done_[2] = {nullptr, nullptr};
  bool branch_ = false;  // total_eager is capturing with branches (near() puts its tile on side_[1])
  void ensure_side();
  DevBuf graph_out_;  // the graph writes here; each replay copies into the caller's arrays

  VertAccel va_;
  HorizAccel ha_;
  DevBuf nu_grid_, nu_partial_, nu_lines_;
  FftPlans fft_;  // this plan's own cuFFT handles (its device, its work areas)
  bool horiz_accel(const Family& f, const Opts& o, periwave::ApplyPath path) const;
  void ensure_horiz_accel(double inner_eps);
  size_t horiz_coeff_len() const;

  void build_families();
  int s2pw_chunks(size_t ns, int modes, int k) const;
  NearKind near_args(const DevSys& s, const Opts& o, const DevOut& out, bool single, double shx, double shy,
                     bool identity, NearArgs& a) const;
  // a vertical scalar family that takes the NUFFT route on this path
  bool vert_accel(const Family& f, const Opts& o, periwave::ApplyPath path) const;
  void ensure_vert_accel(double inner_eps);
  double inner_eps(const Opts& o) const;
  SpreadArgs vert_spread_args(const DevSys& s, bool sources) const;
};

}  // namespace pwb
