// Device plan and orchestration of one apply (host side of the engine).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <vector>

#include "periwave/periwave.hpp"
#include "pw_engine.cuh"

namespace pwb {

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
  ModeTable table() const;
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
  size_t coeff_size(const Opts& o) const;
  void source_pass(const DevSys& s, const Opts& o, double* coeff);
  void target_pass(const DevSys& s, const Opts& o, const double* coeff, const DevOut& out);
  // adds every near image (fused) or one image (single shift)
  void near(const DevSys& s, const Opts& o, const DevOut& out, bool single, double shx, double shy, bool identity);
  // full pipeline on device pointers; returns the accelerated flag
  bool total(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images);

  std::mutex& mutex() { return mu_; }
  // device time (ms) of the last call's phases: [validate+far, near]
  void phase_ms(double* far_ms, double* near_ms);

  // staging for host-memory calls
  DevBuf stage[8];
  PinnedBuf pin;

 private:
  const periwave::Periodizer& pz_;
  int device_ = 0;
  int sms_ = 148;
  cudaStream_t stream_ = nullptr;
  std::vector<std::unique_ptr<Family>> fams_;
  DevBuf s2pw_partial_, coeff_ws_, A_, B_, m0_, near_partial_, flag_, red_m_, red_c_, red_out_;
  PinnedBuf host_checks_;
  DevBuf sym_fx_, sym_rows_;
  PinnedBuf sym_rows_host_;
  std::mutex mu_;
  cudaEvent_t ev_[4] = {nullptr, nullptr, nullptr, nullptr};
  bool far_timed_ = false, near_timed_ = false;

  void build_families();
  int s2pw_chunks(size_t ns, int modes, int k) const;
};

}  // namespace pwb
