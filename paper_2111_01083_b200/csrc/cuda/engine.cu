// Device plan (periodizer tables uploaded once per device) and the
// orchestration of apply_far / total_field / accumulate on device memory.
// Mirrors the control flow of /root/reference/proj/src/apply.cpp:417-556.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.hpp"
#include "nufft.hpp"
#include "pw_math.cuh"

namespace pwb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

void throw_internal(const char* what) { throw InternalFailure(what); }

namespace {
std::atomic<long> g_launches{0};
std::atomic<unsigned long> g_buffer_epoch{0};
}
void count_launches(long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long launch_count() { return g_launches.load(std::memory_order_relaxed); }
unsigned long buffer_epoch() { return g_buffer_epoch.load(std::memory_order_acquire); }

DevBuf::~DevBuf() {
  if (p_) cudaFree(p_);
}

void* DevBuf::ensure(size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (bytes > n_) {
    if (p_) cuda_check(cudaFree(p_), "cudaFree");
    p_ = nullptr;
    n_ = 0;
    g_buffer_epoch.fetch_add(1, std::memory_order_acq_rel);
    cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
    n_ = bytes;
  }
  return p_;
}

PinnedBuf::~PinnedBuf() {
  if (p_) cudaFreeHost(p_);
}

void* PinnedBuf::ensure(size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (bytes > n_) {
    if (p_) cuda_check(cudaFreeHost(p_), "cudaFreeHost");
    p_ = nullptr;
    n_ = 0;
    g_buffer_epoch.fetch_add(1, std::memory_order_acq_rel);
    cuda_check(cudaMallocHost(&p_, bytes), "cudaMallocHost");
    n_ = bytes;
  }
  return p_;
}

using periwave::ErrorCode;
using periwave::require;

Kind kind_of(const periwave::Periodizer& pz) {  // apply.cpp:20-26
  if (pz.multipole_order >= 1) return Kind::Multipole;
  if (pz.pde == periwave::Pde::Stokes || pz.pde == periwave::Pde::ModStokes) return Kind::Velocity;
  return Kind::Scalar;
}

NearKind near_kind_of(const periwave::Periodizer& pz, bool with_pressure, bool with_gradient) {
  const Kind kind = kind_of(pz);
  if (kind == Kind::Multipole) return NearKind::Multipole;
  if (pz.dlp) return NearKind::Stresslet;
  if (kind == Kind::Velocity)
    return pz.pde == periwave::Pde::Stokes ? (with_pressure ? NearKind::StokesP : NearKind::Stokes)
                                           : (with_pressure ? NearKind::ModStokesP : NearKind::ModStokes);
  if (pz.pde == periwave::Pde::ModHelmholtz) return with_gradient ? NearKind::ModHelmGrad : NearKind::ModHelm;
  return NearKind::Laplace;
}

ModeTable Family::table() const {
  ModeTable t;
  t.phase = static_cast<const double*>(phase.get());
  t.decay_t = static_cast<const double*>(decay_t.get());
  t.decay_s = static_cast<const double*>(decay_s.get());
  t.shift_t = static_cast<const double*>(shift_t.get());
  t.shift_s = static_cast<const double*>(shift_s.get());
  t.axis = static_cast<const int*>(axis.get());
  t.count = count;
  return t;
}

namespace {

template <class T>
void upload(DevBuf& b, const std::vector<T>& v) {
  T* p = b.as<T>(v.size());
  if (!v.empty()) cuda_check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
}

struct HostModes {
  std::vector<double> phase, dt, ds, st, ss;
  std::vector<int> axis;
  void add(const periwave::ModeSet& m) {
    for (size_t r = 0; r < m.size(); ++r) {
      phase.push_back(m.phase[r]);
      dt.push_back(m.decay_t[r]);
      ds.push_back(m.decay_s[r]);
      st.push_back(m.shift_t[r]);
      ss.push_back(m.shift_s[r]);
      axis.push_back(m.axis == periwave::Axis::Horizontal ? 1 : 0);
    }
  }
  void to(Family& f) {
    f.count = static_cast<int>(phase.size());
    upload(f.phase, phase);
    upload(f.decay_t, dt);
    upload(f.decay_s, ds);
    upload(f.shift_t, st);
    upload(f.shift_s, ss);
    upload(f.axis, axis);
  }
};

void push_c(std::vector<double>& v, periwave::cplx c) {
  v.push_back(c.real());
  v.push_back(c.imag());
}
void push_m(std::vector<double>& v, const periwave::Mat2c& m) {
  push_c(v, m.a11);
  push_c(v, m.a12);
  push_c(v, m.a21);
  push_c(v, m.a22);
}

void require_vertical_m0(const periwave::ModeSet& m, bool has_m0) {
  require(!has_m0 || m.axis == periwave::Axis::Vertical || m.size() == 0, ErrorCode::Unsupported,
          "rank-one m0 terms are supported on vertical parts only");
}

__global__ void m0_kernel(const double* mom, int ia, int ib, double a00, double a01, double a10, double a11, int ko,
                          double* out) {
  if (threadIdx.x != 0) return;
  const double u = mom[ia], v = mom[ib];
  out[0] = a00 * u + a01 * v;
  out[1] = 0.0;
  if (ko == 2) {
    out[2] = a10 * u + a11 * v;
    out[3] = 0.0;
  }
}

}  // namespace

Plan::Plan(const periwave::Periodizer& pz, int device) : pz_(pz), device_(device) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device_), "sm count");
  // A blocking stream: it orders after work the caller queued on the legacy default
  // stream (e.g. a torch copy of the inputs), so "no stream given" is always safe.
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamDefault), "stream");
  build_families();
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "event");
  flag_.ensure(sizeof(int));
  host_checks_.ensure(64 * sizeof(double));
}

Plan::~Plan() {
  if (cudaGetDevice(&restore_.prev) != cudaSuccess) restore_.prev = -1;
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);  // nothing in flight when the FFT plans and buffers go
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (capture_stream_) cudaStreamDestroy(capture_stream_);
  for (auto& side : side_)
    if (side) cudaStreamDestroy(side);
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  for (auto& e : side_done_)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
}

void Plan::phase_ms(double* far_ms, double* near_ms) {
  float a = 0.f, b = 0.f;
  if (far_timed_) cuda_check(cudaEventElapsedTime(&a, ev_[0], ev_[1]), "event time");
  if (near_timed_) cuda_check(cudaEventElapsedTime(&b, ev_[2], ev_[3]), "event time");
  *far_ms = far_timed_ ? a : 0.0;
  *near_ms = near_timed_ ? b : 0.0;
}

void Plan::build_families() {
  const Kind kind = kind_of(pz_);
  if (kind != Kind::Velocity) {
    // two scalar families: vertical parts (S, N; the accelerated route is the type-1/2
    // NUFFT, apply.cpp:200-259) and horizontal parts (W, E; type 3 on strips, :269-348)
    for (int axis = 0; axis < 2; ++axis) {
      auto f = std::make_unique<Family>();
      f->kind = FamilyKind::Scalar;
      f->ws = kind == Kind::Multipole ? WeightSet::Coef : WeightSet::Charge;
      f->ko = 1;
      f->axis_group = axis;
      HostModes hm;
      std::vector<double> diag;
      double m0sum = 0.0;
      bool any_m0 = false;
      for (const auto& p : pz_.scalar_parts) {
        require(p.diag.size() == p.modes.size(), ErrorCode::LengthMismatch, "scalar part diag/mode size mismatch");
        require_vertical_m0(p.modes, p.has_m0);
        const int pa = p.modes.axis == periwave::Axis::Horizontal ? 1 : 0;
        if (pa != axis) continue;
        hm.add(p.modes);
        f->part_sizes.push_back(static_cast<int>(p.modes.size()));
        for (const auto& c : p.diag) push_c(diag, c);
        if (p.has_m0) {
          any_m0 = true;
          m0sum += p.m0_coef;
        }
      }
      hm.to(*f);
      upload(f->t[0], diag);
      f->host_phase = hm.phase;
      if (any_m0 && kind == Kind::Scalar) {
        f->has_lin = true;
        f->ia = 0;
        f->ib = 0;
        f->mlin[0] = m0sum;
      }
      fams_.push_back(std::move(f));
    }
    return;
  }
  if (!pz_.block_parts.empty()) {
    auto f = std::make_unique<Family>();
    f->kind = FamilyKind::Block;
    f->ko = 2;
    HostModes hm;
    std::vector<double> da, db;
    std::vector<int> tt;
    bool any_three = false, any_m0 = false;
    double msum[4] = {0, 0, 0, 0};
    for (const auto& p : pz_.block_parts) {
      require(p.diag_a.size() == p.modes.size(), ErrorCode::LengthMismatch, "block part diag/mode size mismatch");
      require(!p.three_term || p.diag_b.size() == p.modes.size(), ErrorCode::LengthMismatch,
              "block part diag_b size mismatch");
      require_vertical_m0(p.modes, p.has_m0);
      hm.add(p.modes);
      for (size_t r = 0; r < p.modes.size(); ++r) {
        push_m(da, p.diag_a[r]);
        push_m(db, p.three_term ? p.diag_b[r] : periwave::Mat2c{});
        tt.push_back(p.three_term ? 1 : 0);
      }
      any_three = any_three || p.three_term;
      if (p.has_m0) {
        any_m0 = true;
        msum[0] += p.m0_mat.a11;
        msum[1] += p.m0_mat.a12;
        msum[2] += p.m0_mat.a21;
        msum[3] += p.m0_mat.a22;
      }
    }
    f->ws = any_three ? WeightSet::ForceW : WeightSet::Force;
    hm.to(*f);
    upload(f->t[0], da);
    upload(f->t[1], db);
    upload(f->three_term, tt);
    if (any_m0) {
      f->has_lin = true;
      f->ia = 1;
      f->ib = 2;
      std::memcpy(f->mlin, msum, sizeof msum);
    }
    fams_.push_back(std::move(f));
  }
  if (!pz_.stresslet_parts.empty()) {
    auto f = std::make_unique<Family>();
    f->kind = FamilyKind::Stresslet;
    f->ws = WeightSet::DoubleLayer;
    f->ko = 2;
    HostModes hm;
    std::vector<double> a1, a2, sm, sa, sb, off;
    double csum = 0.0;
    bool any_m0 = false;
    for (const auto& p : pz_.stresslet_parts) {
      const size_t n = p.modes.size();
      require(p.a1.size() == n && p.a2.size() == n && p.smat.size() == n && p.sa.size() == n && p.sb.size() == n &&
                  p.off.size() == n,
              ErrorCode::LengthMismatch, "stresslet part table size mismatch");
      require_vertical_m0(p.modes, p.has_m0);
      hm.add(p.modes);
      for (size_t r = 0; r < n; ++r) {
        push_m(a1, p.a1[r]);
        push_m(a2, p.a2[r]);
        push_m(sm, p.smat[r]);
        push_c(sa, p.sa[r]);
        push_c(sb, p.sb[r]);
        push_c(off, p.off[r]);
      }
      if (p.has_m0) {
        any_m0 = true;
        csum += p.m0_coef;
      }
    }
    hm.to(*f);
    upload(f->t[0], a1);
    upload(f->t[1], a2);
    upload(f->t[2], sm);
    upload(f->t[3], sa);
    upload(f->t[4], sb);
    upload(f->t[5], off);
    if (any_m0) {
      f->has_lin = true;
      f->ia = 3;
      f->ib = 4;
      f->mlin[0] = csum;
      f->mlin[3] = csum;
    }
    fams_.push_back(std::move(f));
  }
  if (!pz_.pressure_parts.empty()) {
    auto f = std::make_unique<Family>();
    f->kind = FamilyKind::Pressure;
    f->ws = WeightSet::Force;
    f->ko = 1;
    f->pressure = true;
    HostModes hm;
    std::vector<double> diag, row;
    bool any_m0 = false;
    double cx = 0.0, cy = 0.0;
    for (const auto& p : pz_.pressure_parts) {
      require(p.diag.size() == p.modes.size() && p.row.size() == p.modes.size(), ErrorCode::LengthMismatch,
              "pressure part table size mismatch");
      require_vertical_m0(p.modes, p.has_m0);
      hm.add(p.modes);
      for (size_t r = 0; r < p.modes.size(); ++r) {
        push_c(diag, p.diag[r]);
        push_c(row, p.row[r].x);
        push_c(row, p.row[r].y);
      }
      if (p.has_m0) {
        any_m0 = true;
        cx += p.m0_coef * p.m0_row.x;
        cy += p.m0_coef * p.m0_row.y;
      }
    }
    hm.to(*f);
    upload(f->t[0], diag);
    upload(f->t[1], row);
    if (any_m0) {
      f->has_cst = true;
      f->ia = 1;
      f->ib = 2;
      f->mcst[0] = cx;
      f->mcst[1] = cy;
    }
    fams_.push_back(std::move(f));
  }
}

int Plan::s2pw_chunks(size_t ns, int modes, int k) const {
  const int mt = k >= 8 ? 1 : 8 / k;
  const int mode_blocks = std::max(1, (modes + mt - 1) / mt);
  long want = (4L * sms_ + mode_blocks - 1) / mode_blocks;
  const long by_src = static_cast<long>(std::max<size_t>(1, ns / 256));  // >= 256 sources per chunk
  want = std::min(want, by_src);
  return static_cast<int>(std::max(1L, std::min(want, 1024L)));
}

periwave::ApplyPath Plan::resolve(const Opts& o, size_t n_src_total, size_t n_tgt_total) const {
  if (o.path != periwave::ApplyPath::Auto) return o.path;
  return periwave::choose_path(pz_, n_src_total, n_tgt_total);
}

bool Plan::vert_accel(const Family& f, const Opts& o, periwave::ApplyPath path) const {
  // the gradient extension needs per-mode derivative symbols: it stays on the direct sweep
  return path == periwave::ApplyPath::Accelerated && f.kind == FamilyKind::Scalar && f.axis_group == 0 &&
         f.count > 0 && !o.with_gradient;
}

bool Plan::horiz_accel(const Family& f, const Opts& o, periwave::ApplyPath path) const {
  // apply.cpp:456-458: the west/east parts accelerate on singly periodic cells only
  return path == periwave::ApplyPath::Accelerated && f.kind == FamilyKind::Scalar && f.axis_group == 1 &&
         f.count > 0 && pz_.cell.periodicity == periwave::Periodicity::Singly && !o.with_gradient;
}

void Plan::ensure_horiz_accel(double eps) {
  const Family& f = *fams_[1];
  const periwave::UnitCell& c = pz_.cell;
  if (!ha_.ready) {
    // interval of the closed cell in x (cell.cpp:66-70 slack) instead of the data span of
    // apply.cpp:275-285: covers every admissible point, and is the same on every rank
    const double ext = (0.5 + 1e-12) * (c.d + std::abs(c.xi));
    ha_.lo = -ext;
    ha_.hi = ext;
    ha_.ymax = (0.5 + 1e-12) * c.eta;
    const double width = ha_.hi - ha_.lo;
    const double margin = 2.0 * c.d - width;  // > 0: |xi| <= d/2 on strips
    const double e = std::max(pz_.eps, 1e-14);
    const double u = 1.0 + 2.0 * margin / width;
    const double rho = u + std::sqrt(u * u - 1.0);
    ha_.mg = std::clamp(static_cast<int>(std::ceil(std::log(1.0 / e) / std::log(rho))) + 2, 4, 64);  // apply.cpp:290
    const periwave::BarycentricGrid g = periwave::make_barycentric_grid(ha_.lo, ha_.hi, ha_.mg);
    for (int k = 0; k < ha_.mg; ++k) {
      ha_.tk[k] = (2.0 * g.nodes[k] - g.lo - g.hi) / (g.hi - g.lo);
      ha_.bw[k] = g.bary_w[k];
    }
    upload(ha_.nodes, g.nodes);
    std::vector<double> neg(f.host_phase.size());
    ha_.lmax = 0.0;
    for (size_t r = 0; r < neg.size(); ++r) {
      neg[r] = -f.host_phase[r];
      ha_.lmax = std::max(ha_.lmax, std::abs(f.host_phase[r]));
    }
    upload(ha_.neg_lam, neg);
    ha_.part_start.assign(1, 0);
    for (int sz : f.part_sizes) ha_.part_start.push_back(ha_.part_start.back() + sz);
    ha_.ready = true;
  }
  if (ha_.eps != eps) {
    const EsSpec s = es_spec(eps);
    ha_.w = s.w;
    ha_.beta = s.beta;
    // source side: x = y_j, s = -lambda (nufft_fast.cpp:505-507)
    ha_.hx1 = periwave::kPi / (2.0 * ha_.lmax);
    ha_.nf1 = static_cast<int>(next_fast_even(2 * static_cast<size_t>(std::ceil(ha_.ymax / ha_.hx1)) + 2 * s.w + 4));
    std::vector<double> fac(f.host_phase.size());
    for (size_t r = 0; r < fac.size(); ++r)
      fac[r] = (2.0 / s.w) / phihat(s, -f.host_phase[r] * 0.5 * s.w * ha_.hx1);
    upload(ha_.fac1, fac);
    // target side: x = lambda_r, s = y_l
    ha_.hx2 = periwave::kPi / (2.0 * ha_.ymax);
    ha_.nf2 = static_cast<int>(next_fast_even(2 * static_cast<size_t>(std::ceil(ha_.lmax / ha_.hx2)) + 2 * s.w + 4));
    require(ha_.nf1 <= (1 << 24) && ha_.nf2 <= (1 << 24), ErrorCode::Unsupported, "type-3 transform extent too large");
    const periwave::GaussRule gl = periwave::gauss_legendre(3 * s.w + 20);
    std::vector<double> amp(gl.nodes.size());
    for (size_t i = 0; i < amp.size(); ++i) {
      const double t = 1.0 - gl.nodes[i] * gl.nodes[i];
      amp[i] = gl.weights[i] * (t <= 0.0 ? 0.0 : std::exp(s.beta * (std::sqrt(t) - 1.0)));
    }
    ha_.ngl = static_cast<int>(amp.size());
    upload(ha_.gl_amp, amp);
    upload(ha_.gl_z, gl.nodes);
    ha_.eps = eps;
  }
}

double Plan::inner_eps(const Opts& o) const {  // apply.cpp:213
  return o.nufft_eps > 0.0 ? o.nufft_eps : std::max(1e-14, 0.01 * pz_.eps);
}

void Plan::ensure_vert_accel(double eps) {
  const Family& f = *fams_[0];
  if (!va_.ready) {
    const periwave::UnitCell& c = pz_.cell;
    const double kx = c.d / (2.0 * periwave::kPi);
    long mmax = 0;  // apply.cpp:206-210
    for (double ph : f.host_phase) mmax = std::max(mmax, std::lround(std::abs(ph) * kx));
    va_.mmax = static_cast<int>(mmax);
    va_.nmodes = static_cast<int>(2 * mmax + 1);
    va_.mg = periwave::interp_nodes_for(pz_.eps);
    require(va_.mg <= 64, ErrorCode::Unsupported, "at most 64 interpolation lines");
    const periwave::BarycentricGrid g = periwave::make_barycentric_grid(-0.5 * c.eta, 0.5 * c.eta, va_.mg);
    va_.lo = g.lo;
    va_.hi = g.hi;
    va_.nodes_host = g.nodes;
    for (int k = 0; k < va_.mg; ++k) {  // quadrature.cpp:291-299 reference coordinates
      va_.tk[k] = (2.0 * g.nodes[k] - g.lo - g.hi) / (g.hi - g.lo);
      va_.bw[k] = g.bary_w[k];
    }
    upload(va_.nodes, g.nodes);
    std::vector<std::vector<int>> buckets(va_.nmodes);
    for (size_t r = 0; r < f.host_phase.size(); ++r)
      buckets[static_cast<size_t>(std::lround(f.host_phase[r] * kx) + mmax)].push_back(static_cast<int>(r));
    std::vector<int> start(1, 0), list;
    for (const auto& b : buckets) {
      list.insert(list.end(), b.begin(), b.end());
      start.push_back(static_cast<int>(list.size()));
    }
    upload(va_.bucket_start, start);
    upload(va_.bucket, list);
    va_.ready = true;
  }
  if (va_.eps != eps) {
    const EsSpec s = es_spec(eps);
    va_.w = s.w;
    va_.beta = s.beta;
    va_.nf = static_cast<int>(grid_size_for_modes(static_cast<size_t>(va_.nmodes), s));
    upload(va_.fac, deconv_factors(s, static_cast<size_t>(va_.nf), static_cast<size_t>(va_.nmodes)));
    va_.eps = eps;
  }
}

size_t Plan::coeff_size(const Opts& o, periwave::ApplyPath path) {
  size_t n = 0;
  for (const auto& f : fams_) {
    if (f->pressure && !o.with_pressure) continue;
    if (vert_accel(*f, o, path)) {
      ensure_vert_accel(inner_eps(o));
      n += static_cast<size_t>(va_.mg) * va_.nmodes * 2;  // F lines (type-1 output per Legendre line)
    } else if (horiz_accel(*f, o, path)) {
      ensure_horiz_accel(inner_eps(o));
      n += static_cast<size_t>(ha_.mg) * f->count * 2;  // F_k[r] (type-3 output per line and mode)
    } else {
      n += static_cast<size_t>(f->count) * weight_count(f->ws) * 2;
    }
  }
  return n + kMoments + 3;  // moments, padded to a multiple of 8 bytes * 8
}

void Plan::validate(const DevSys& s, const Opts& o, bool far_checks, bool neutrality) {
  const Kind kind = kind_of(pz_);
  // apply.cpp:350-364 + cell.cpp:84-91: the strength arrays the kind needs
  if (kind == Kind::Multipole)
    require(s.ns == 0 || s.coef, ErrorCode::LengthMismatch, "multipole apply requires one complex coefficient per source");
  else if (pz_.dlp)
    require(s.ns == 0 || (s.f && s.nrm), ErrorCode::LengthMismatch,
            "double-layer apply requires a force vector and a unit normal per source");
  else if (kind == Kind::Velocity)
    require(s.ns == 0 || s.f, ErrorCode::LengthMismatch, "velocity apply requires one force vector per source");
  else
    require(s.ns == 0 || s.q, ErrorCode::LengthMismatch, "scalar apply requires one charge per source");
  if (far_checks) {
    require(!o.with_pressure || !pz_.pressure_parts.empty(), ErrorCode::Unsupported,
            "pressure output is not available for this periodizer");
  } else {
    require(!o.with_pressure || kind == Kind::Velocity, ErrorCode::Unsupported,
            "pressure output is not available for this periodizer");
    require(!(o.with_pressure && pz_.dlp), ErrorCode::Unsupported,
            "pressure output is not available for the double-layer kernel");
  }
  require(!o.with_gradient || (kind == Kind::Scalar && pz_.pde == periwave::Pde::ModHelmholtz), ErrorCode::Unsupported,
          "gradient output is available for the modified Helmholtz scalar kernel");
  cudaStream_t st = stream_for(o);
  ReduceArgs ra;
  ra.src = s.src;
  ra.ns = s.ns;
  ra.q = s.q;
  ra.vec = s.f;
  ra.coef = s.coef;
  ra.nrm = s.nrm;
  ra.tgt = far_checks ? s.tgt : nullptr;
  ra.nt = far_checks ? s.nt : 0;
  ra.d = pz_.cell.d;
  ra.xi = pz_.cell.xi;
  ra.eta = pz_.cell.eta;
  double* bm = red_m_.as<double>(kReduceBlocks * kMoments);
  double* bc = red_c_.as<double>(kReduceBlocks * kChecks);
  double* outv = red_out_.as<double>(kMoments + kChecks);
  const int rb = reduce_blocks(std::max(ra.ns, ra.nt));
  launch_reduce(ra, bm, bc, rb, st);
  launch_sum_blocks(bc, rb, kChecks, outv + kMoments, st);
  // the block moments of the same sources: source_pass may reuse them (moments_ready)
  moment_blocks_ = rb;
  cuda_check(cudaGetLastError(), "validate launch");
  const double* h = static_cast<double*>(host_checks_.ensure(64 * sizeof(double)));
  cuda_check(cudaMemcpyAsync(const_cast<double*>(h), outv + kMoments, kChecks * sizeof(double), cudaMemcpyDeviceToHost,
                             st),
             "D2H checks");
  const bool neutral = pz_.requires_neutrality && neutrality;
  auto check = [h, far_checks, neutral, kind] {
    if (far_checks)
      require(h[0] == 0.0, ErrorCode::OutOfInterval, "source or target point outside the closed unit cell");
    require(h[1] == 0.0, ErrorCode::NonUnitNormal, "stresslet normals must be unit vectors");
    if (!neutral) return;  // apply.cpp:365-392
    if (kind == Kind::Multipole)
      require(std::hypot(h[7], h[8]) <= 1e-12 * h[9], ErrorCode::NotNeutral,
              "this periodizer requires coefficients summing to zero");
    else if (kind == Kind::Velocity)
      require(std::hypot(h[4], h[5]) <= 1e-12 * h[6], ErrorCode::NotNeutral,
              "this periodizer requires forces summing to zero");
    else
      require(std::abs(h[2]) <= 1e-12 * h[3], ErrorCode::NotNeutral,
              "this periodizer requires charges summing to zero");
  };
  if (defer_) {
    pending_.push_back(check);
    return;
  }
  cuda_check(cudaStreamSynchronize(st), "validate sync");
  check();
}

SpreadArgs Plan::vert_spread_args(const DevSys& s, bool sources) const {
  SpreadArgs a;
  a.pos = PosKind::WrappedX;  // x~ = -wrap(x) 2 pi / d (apply.cpp:219, :247)
  a.pts = sources ? s.src : s.tgt;
  a.n = sources ? s.ns : s.nt;
  a.d = pz_.cell.d;
  a.kx = 2.0 * periwave::kPi / pz_.cell.d;
  a.nf = va_.nf;
  a.h = 2.0 * periwave::kPi / static_cast<double>(va_.nf);
  a.w = va_.w;
  a.beta = va_.beta;
  a.lines = va_.mg;
  a.bary.lo = va_.lo;
  a.bary.hi = va_.hi;
  a.bary.m = va_.mg;
  for (int k = 0; k < va_.mg; ++k) {
    a.bary.tk[k] = va_.tk[k];
    a.bary.bw[k] = va_.bw[k];
  }
  a.bary_axis = 0;  // Legendre lines in y
  return a;
}

void Plan::source_pass(const DevSys& s, const Opts& o, double* coeff, periwave::ApplyPath path, bool moments_ready,
                       cudaEvent_t moments_after) {
  cudaStream_t st = stream_for(o);
  size_t off = 0;
  for (const auto& fp : fams_) {
    Family& f = *fp;
    if (f.pressure && !o.with_pressure) continue;
    const int k = weight_count(f.ws);
    f.raw_offset = off;
    if (vert_accel(f, o, path)) {
      // apply.cpp:216-228: c_jk = gamma_k(y_j) q_j spread on each Legendre line, type 1 per line
      ensure_vert_accel(inner_eps(o));
      SpreadArgs a = vert_spread_args(s, true);
      a.c = f.ws == WeightSet::Coef ? reinterpret_cast<const double*>(s.coef) : s.q;
      a.cplx = f.ws == WeightSet::Coef ? 1 : 0;
      double* grid = nu_grid_.as<double>(static_cast<size_t>(va_.mg) * va_.nf * 2);
      launch_spread(a, grid, nu_partial_, sms_, st);
      fft_.exec(grid, va_.nf, va_.mg, +1, st);
      launch_deconv(grid, va_.mg, va_.nf, va_.nmodes, static_cast<const double*>(va_.fac.get()), coeff + off, st);
      off += static_cast<size_t>(va_.mg) * va_.nmodes * 2;
      continue;
    }
    if (horiz_accel(f, o, path)) {
      // apply.cpp:313-319: F_k[r] = sum_j gamma_k(x_j) q_j e^{-i lambda_r y_j} (type 3 per line);
      // the spread depends on neither the part nor the mode, so it is done once for all lines
      ensure_horiz_accel(inner_eps(o));
      SpreadArgs a;
      a.pos = PosKind::PointY;
      a.pts = s.src;
      a.n = s.ns;
      a.c = f.ws == WeightSet::Coef ? reinterpret_cast<const double*>(s.coef) : s.q;
      a.cplx = f.ws == WeightSet::Coef ? 1 : 0;
      a.open = 1;
      a.inv_h = 1.0 / ha_.hx1;
      a.nf = ha_.nf1;
      a.w = ha_.w;
      a.beta = ha_.beta;
      a.lines = ha_.mg;
      a.bary.lo = ha_.lo;
      a.bary.hi = ha_.hi;
      a.bary.m = ha_.mg;
      for (int k = 0; k < ha_.mg; ++k) {
        a.bary.tk[k] = ha_.tk[k];
        a.bary.bw[k] = ha_.bw[k];
      }
      a.bary_axis = 1;  // Legendre lines in x
      double* grid = nu_grid_.as<double>(static_cast<size_t>(ha_.mg) * ha_.nf1 * 2);
      launch_spread(a, grid, nu_partial_, sms_, st);
      launch_exact_lines(grid, ha_.mg, ha_.nf1, static_cast<const double*>(ha_.neg_lam.get()), f.count, ha_.hx1,
                         static_cast<const double*>(ha_.fac1.get()), coeff + off, st);
      off += static_cast<size_t>(ha_.mg) * f.count * 2;
      continue;
    }
    const size_t len = static_cast<size_t>(f.count) * k * 2;
    if (f.count > 0) {
      // small problems: one chunk, one mode per block, the kernel writes the raw sums
      const bool narrow = s.ns <= kS2pwNarrowSources;
      const int chunks = (s.ns == 0 || narrow) ? 1 : s2pw_chunks(s.ns, f.count, k);
      S2pwArgs a;
      a.narrow = narrow ? 1 : 0;
      a.modes = f.table();
      a.src = s.src;
      a.q = s.q;
      a.vec = f.ws == WeightSet::Coef ? s.coef : s.f;
      a.nrm = s.nrm;
      a.ns = s.ns;
      a.chunks = chunks;
      a.per_chunk = (s.ns + chunks - 1) / chunks;
      if (chunks == 1) {
        a.partial = coeff + off;
        launch_s2pw(f.ws, a, st);
      } else {
        a.partial = s2pw_partial_.as<double>(static_cast<size_t>(chunks) * len);
        launch_s2pw(f.ws, a, st);
        launch_chunk_sum(a.partial, chunks, len, coeff + off, st);
      }
    }
    off += len;
  }
  // rank-one moments (apply.cpp:68-78, :108-117, :140-146, :179-191). Right after a
  // validation of the same system its block moments are already there (the moments used
  // by the families depend on the sources only; the charge moment only when the kind reads
  // charges, which is the only case validate's charge sums can differ in).
  double* bm = red_m_.as<double>(kReduceBlocks * kMoments);
  int rb = moment_blocks_;
  // a validation branch owns red_m_ / red_c_ until its event (reused or overwritten below)
  if (moments_after) cuda_check(cudaStreamWaitEvent(st, moments_after, 0), "moments wait");
  if (!(moments_ready && (kind_of(pz_) == Kind::Scalar || s.q == nullptr))) {
    ReduceArgs ra;
    ra.src = s.src;
    ra.ns = s.ns;
    ra.q = kind_of(pz_) == Kind::Scalar ? s.q : nullptr;
    ra.vec = s.f;
    ra.nrm = s.nrm;
    double* bc = red_c_.as<double>(kReduceBlocks * kChecks);
    rb = reduce_blocks(s.ns);
    launch_reduce(ra, bm, bc, rb, st);
  }
  launch_sum_blocks(bm, rb, kMoments, coeff + off, st);
  cuda_check(cudaGetLastError(), "source pass launch");
}

bool Plan::target_pass(const DevSys& s, const Opts& o, const double* coeff, const DevOut& out,
                       periwave::ApplyPath path) {
  cudaStream_t st = stream_for(o);
  const Kind kind = kind_of(pz_);
  bool accelerated = false;
  // zero the outputs this kind produces, then every family accumulates
  if (s.nt > 0) {
    if (kind == Kind::Scalar) cuda_check(cudaMemsetAsync(out.scalar, 0, s.nt * sizeof(double), st), "memset");
    if (kind == Kind::Multipole)
      cuda_check(cudaMemsetAsync(out.complex_scalar, 0, 2 * s.nt * sizeof(double), st), "memset");
    if (kind == Kind::Velocity) cuda_check(cudaMemsetAsync(out.velocity, 0, 2 * s.nt * sizeof(double), st), "memset");
    if (o.with_pressure) cuda_check(cudaMemsetAsync(out.pressure, 0, s.nt * sizeof(double), st), "memset");
    if (o.with_gradient) cuda_check(cudaMemsetAsync(out.gradient, 0, 2 * s.nt * sizeof(double), st), "memset");
  }
  size_t off = 0;
  const size_t mom_off = coeff_size(o, path) - kMoments - 3;
  for (const auto& fp : fams_) {
    Family& f = *fp;
    if (f.pressure && !o.with_pressure) continue;
    const int k = weight_count(f.ws);
    const bool haccel = horiz_accel(f, o, path);
    if (haccel) {
      // apply.cpp:321-346 per part: mixing, type 3 lambda -> y per line, barycentric sum in x
      ensure_horiz_accel(inner_eps(o));
      const int nr_all = f.count;
      for (size_t p = 0; p + 1 < ha_.part_start.size() && s.nt > 0; ++p) {
        const int r0 = ha_.part_start[p], nr = ha_.part_start[p + 1] - r0;
        if (nr == 0) continue;
        HmixArgs ma;
        ma.nr = nr;
        ma.lines = ha_.mg;
        ma.stride = nr_all;
        ma.f_off = r0;
        ma.decay_s = static_cast<const double*>(f.decay_s.get()) + r0;
        ma.shift_s = static_cast<const double*>(f.shift_s.get()) + r0;
        ma.decay_t = static_cast<const double*>(f.decay_t.get()) + r0;
        ma.shift_t = static_cast<const double*>(f.shift_t.get()) + r0;
        ma.diag = static_cast<const double*>(f.t[0].get()) + 2 * r0;
        ma.nodes = static_cast<const double*>(ha_.nodes.get());
        ma.lam = static_cast<const double*>(f.phase.get()) + r0;
        ma.inv_h = 1.0 / ha_.hx2;
        ma.nf = ha_.nf2;
        ma.w = ha_.w;
        ma.beta = ha_.beta;
        double* Aw = nu_lines_.as<double>(static_cast<size_t>(ha_.mg) * nr * 2);
        launch_hmix(ma, coeff + off, Aw, st);
        double* grid = nu_grid_.as<double>(static_cast<size_t>(ha_.mg) * ha_.nf2 * 2);
        launch_lam_spread(ma, Aw, grid, st);
        HtgtArgs ta2;
        ta2.nt = s.nt;
        ta2.tgt = s.tgt;
        ta2.lo = ha_.lo;
        ta2.hi = ha_.hi;
        ta2.lines = ha_.mg;
        for (int kk = 0; kk < ha_.mg; ++kk) {
          ta2.tk[kk] = ha_.tk[kk];
          ta2.bw[kk] = ha_.bw[kk];
        }
        ta2.hx = ha_.hx2;
        ta2.nf = ha_.nf2;
        ta2.w = ha_.w;
        ta2.ngl = ha_.ngl;
        ta2.gl_amp = static_cast<const double*>(ha_.gl_amp.get());
        ta2.gl_z = static_cast<const double*>(ha_.gl_z.get());
        launch_htarget(ta2, grid, kind == Kind::Multipole ? nullptr : out.scalar,
                       kind == Kind::Multipole ? out.complex_scalar : nullptr, st);
      }
      accelerated = true;
      off += static_cast<size_t>(ha_.mg) * f.count * 2;
      continue;
    }
    const bool accel = vert_accel(f, o, path);
    const size_t len = accel ? static_cast<size_t>(va_.mg) * va_.nmodes * 2 : static_cast<size_t>(f.count) * k * 2;
    double* A = A_.as<double>(static_cast<size_t>(std::max(f.count, 1)) * f.ko * 2);
    double* B = B_.as<double>(static_cast<size_t>(std::max(f.count, 1)) * f.ko * 2);
    double* m0 = m0_.as<double>(8);
    PrepArgs pa;
    pa.kind = f.kind;
    pa.count = f.count;
    pa.k = k;
    pa.raw = coeff + off;
    for (int i = 0; i < 6; ++i) {
      const double* tp = static_cast<const double*>(f.t[i].get());
      switch (i) {
        case 0: pa.t0 = tp; break;
        case 1: pa.t1 = tp; break;
        case 2: pa.t2 = tp; break;
        case 3: pa.t3 = tp; break;
        case 4: pa.t4 = tp; break;
        default: pa.t5 = tp; break;
      }
    }
    pa.three_term = static_cast<const int*>(f.three_term.get());
    pa.A = A;
    pa.B = B;
    if (!accel) launch_prep(pa, st);
    if (f.has_lin || f.has_cst) {
      const double* mv = f.has_lin ? f.mlin : nullptr;
      if (f.has_lin)
        m0_kernel<<<1, 32, 0, st>>>(coeff + mom_off, f.ia, f.ib, mv[0], mv[1], mv[2], mv[3], f.ko, m0);
      else
        m0_kernel<<<1, 32, 0, st>>>(coeff + mom_off, f.ia, f.ib, f.mcst[0], f.mcst[1], 0.0, 0.0, f.ko, m0);
      count_launches(1);
    }
    Pw2tArgs ta;
    ta.modes = f.table();
    ta.A = A;
    ta.B = (f.kind == FamilyKind::Block || f.kind == FamilyKind::Stresslet) ? B : nullptr;
    ta.tgt = s.tgt;
    ta.nt = s.nt;
    ta.ko = f.ko;
    ta.gradient = (f.kind == FamilyKind::Scalar && o.with_gradient) ? 1 : 0;
    ta.m0_lin = f.has_lin ? m0 : nullptr;
    ta.m0_const = f.has_cst ? m0 : nullptr;
    ta.accumulate = 1;
    if (f.kind == FamilyKind::Pressure) {
      ta.out_re = out.pressure;
    } else if (kind == Kind::Multipole) {
      ta.out_cplx = out.complex_scalar;
    } else if (kind == Kind::Velocity) {
      ta.out_re = out.velocity;
    } else {
      ta.out_re = out.scalar;
      ta.out_grad = out.gradient;
    }
    if (accel) {
      // rank-one m0 terms stay direct (apply.cpp:462); no plane-wave modes in this launch
      ta.modes.count = 0;
      if (f.has_lin) launch_pw2t(ta, st);
      if (s.nt > 0) {
        // apply.cpp:230-258: mode mixing, one type 2 per line, barycentric sum over lines
        MixArgs ma;
        ma.nmodes = va_.nmodes;
        ma.lines = va_.mg;
        ma.bucket_start = static_cast<const int*>(va_.bucket_start.get());
        ma.bucket = static_cast<const int*>(va_.bucket.get());
        ma.decay_s = static_cast<const double*>(f.decay_s.get());
        ma.shift_s = static_cast<const double*>(f.shift_s.get());
        ma.decay_t = static_cast<const double*>(f.decay_t.get());
        ma.shift_t = static_cast<const double*>(f.shift_t.get());
        ma.diag = static_cast<const double*>(f.t[0].get());
        ma.nodes = static_cast<const double*>(va_.nodes.get());
        double* G = nu_lines_.as<double>(static_cast<size_t>(va_.mg) * va_.nmodes * 2);
        launch_mix(ma, coeff + off, G, st);
        double* grid = nu_grid_.as<double>(static_cast<size_t>(va_.mg) * va_.nf * 2);
        launch_precorrect(G, va_.mg, va_.nf, va_.nmodes, static_cast<const double*>(va_.fac.get()), grid, st);
        fft_.exec(grid, va_.nf, va_.mg, -1, st);
        const SpreadArgs a = vert_spread_args(s, false);
        launch_interp(a, grid, kind == Kind::Multipole ? nullptr : out.scalar,
                      kind == Kind::Multipole ? out.complex_scalar : nullptr, true, st);
      }
      accelerated = true;
    } else {
      launch_pw2t(ta, st);
    }
    off += len;
  }
  cuda_check(cudaGetLastError(), "target pass launch");
  return accelerated;
}

double screen_cutoff(double eps, int images, size_t ns, bool grad);
bool near_screened(NearKind nk, const NearArgs& a);
bool prod_form(const periwave::Periodizer& pz, NearKind nk, NearArgs& a, size_t n);

NearKind Plan::near_args(const DevSys& s, const Opts& o, const DevOut& out, bool single, double shx, double shy,
                         bool identity, NearArgs& a) const {
  const Kind kind = kind_of(pz_);
  NearKind nk;
  a.tgt = s.tgt;
  a.nt = s.nt;
  a.src = s.src;
  a.ns = s.ns;
  a.q = s.q;
  a.nrm = s.nrm;
  a.vec = s.f;
  a.beta = pz_.beta;
  a.beta2 = pz_.beta * pz_.beta;
  a.xcut2 = 64.0 * 64.0;  // K_0(x) < 3e-29 beyond; screened kinds refine it below (screen_cutoff)
  // precision tier of the near tiles (pw_math.cuh log_pos_k, k01_tile): the reduced tier
  // keeps |error| <= ~3e-13 per pair-log and <= 6e-14 relative per Bessel value, >= 1.5
  // orders below eps for eps >= 1e-11 (the reference's eps bounds the far truncation);
  // the full tier is ~1 ulp. PWB_FULL_PRECISION forces the full tier (tests).
  a.lowp = (pz_.eps >= 1e-11 && std::getenv("PWB_FULL_PRECISION") == nullptr) ? 1 : 0;
  // coarse Bessel tier of the screened tiles: <= ~1e-11 relative per K0 / K1 (pinned by
  // test_hot_tile_bessel_coarse_tier), for eps >= 1e-10 -- measured 9.8e-13 on c2 (eps 1e-10,
  // bar 1e-9) and 7e-12 on c5 (eps 1e-8, bar 1e-7), profiles/r1b_parity.json;
  // PWB_NO_COARSE keeps the reduced tier, PWB_COARSE_EPS moves the threshold (A/B)
  const char* ce = std::getenv("PWB_COARSE_EPS");
  const double coarse_eps = ce ? std::atof(ce) : 1e-10;
  if (a.lowp && pz_.eps >= coarse_eps && std::getenv("PWB_NO_COARSE") == nullptr) a.lowp = 2;
  // coarse table log of the symmetric Laplace / Stokeslet tiles: <= 9.1e-13 absolute per
  // pair-log, two orders below eps >= 1e-10 (c4: eps = 1e-10; c3: 1e-8)
  a.coarse_log = (a.lowp && pz_.eps >= 1e-10 && std::getenv("PWB_NO_COARSE") == nullptr) ? 1 : 0;
  a.cull = std::getenv("PWB_NO_CULL") == nullptr ? 1 : 0;  // A/B and the exactness test only
  if (kind == Kind::Multipole) {
    nk = NearKind::Multipole;
    a.vec = s.coef;
    a.order = pz_.multipole_order;
    a.screened = pz_.pde == periwave::Pde::ModHelmholtz ? 1 : 0;
    a.out0 = out.complex_scalar;
    a.nout0 = 2;
  } else if (pz_.dlp) {
    nk = NearKind::Stresslet;
    a.out0 = out.velocity;
    a.nout0 = 2;
  } else if (kind == Kind::Velocity) {
    const bool p = o.with_pressure;
    nk = pz_.pde == periwave::Pde::Stokes ? (p ? NearKind::StokesP : NearKind::Stokes)
                                          : (p ? NearKind::ModStokesP : NearKind::ModStokes);
    a.ms_scale = pz_.pde == periwave::Pde::ModStokes ? 1.0 / (2.0 * periwave::kPi * a.beta2) : 0.0;
    a.out0 = out.velocity;
    a.nout0 = 2;
    if (p) {
      a.out1 = out.pressure;
      a.nout1 = 1;
    }
  } else if (pz_.pde == periwave::Pde::ModHelmholtz) {
    nk = o.with_gradient ? NearKind::ModHelmGrad : NearKind::ModHelm;
    a.out0 = out.scalar;
    a.nout0 = 1;
    if (o.with_gradient) {
      a.out1 = out.gradient;
      a.nout1 = 2;
    }
  } else {
    nk = NearKind::Laplace;
    a.out0 = out.scalar;
    a.nout0 = 1;
  }
  if (single) {
    a.nxi = 1;
    a.nrow = 1;
    a.shx[0] = shx;
    a.shy[0] = shy;
    a.id_img = identity ? 0 : -1;
  } else {
    const periwave::UnitCell& c = pz_.cell;
    if (c.periodicity == periwave::Periodicity::Doubly) {
      a.nxi = 2 * c.m0 + 1;
      a.nrow = 3;
      for (int n = -1; n <= 1; ++n) {
        a.shy[n + 1] = n * c.eta;
        for (int m = -c.m0; m <= c.m0; ++m) a.shx[(n + 1) * a.nxi + (m + c.m0)] = m * c.d + n * c.xi;
      }
      a.id_img = 1 * a.nxi + c.m0;
      a.unskewed = c.xi == 0.0 ? 1 : 0;
    } else {
      a.nxi = 3;
      a.nrow = 1;
      a.shy[0] = 0.0;
      for (int m = -1; m <= 1; ++m) a.shx[m + 1] = m * c.d;
      a.id_img = 1;
    }
  }
  if (nk == NearKind::ModHelm || nk == NearKind::ModHelmGrad) {
    const double xc = screen_cutoff(pz_.eps, a.nxi * a.nrow, s.ns, nk == NearKind::ModHelmGrad);
    // round x_c^2 up to a zero low word: the tiles compare high words on the integer pipe
    // (pw_math.cuh lt_hi), exact for such a bound
    a.xcut2 = pwk::hi_lo(pwk::hi_of(xc * xc) + (pwk::lo_of(xc * xc) != 0u ? 1 : 0), 0u);
    // per-tile-pair Chebyshev K0 of the symmetric tile (pw_math.cuh cheb_fit_k0): relative
    // error <= 1e-3 eps per pair, in the coarse tier (eps >= 1e-10); PWB_NO_CHEB: off (A/B)
    if (nk == NearKind::ModHelm && a.lowp == 2 && std::getenv("PWB_NO_CHEB") == nullptr) {
      a.cheb_tol = 1e-3 * pz_.eps;
      a.inv_beta2 = 1.0 / a.beta2;
    }
  }
  return nk;
}

// Screening cut-off of the modified-Helmholtz near tiles: pairs with x = beta r >= x_c
// are skipped, x_c the smallest x in [2, 64] with K0(x) <= 1e-3 eps / (images * N_S)
// (K1 for the gradient, with a factor 2 of margin). Every target then loses at most
// 1e-3 eps max|q| / 2pi in total -- a thousandth of eps times the field of one unit
// source at beta r ~ 0.6 (K0 = 1 / 2pi scale) -- while the parity bar is 10 eps
// relative. The reference sums every pair to GSL's underflow (x ~ 700); K0(64) ~ 3e-29,
// the previous fixed cut-off, is the upper end. PWB_KCUT=<x> overrides (A/B, tests).
double screen_cutoff(double eps, int images, size_t ns, bool grad) {
  if (const char* e = std::getenv("PWB_KCUT")) return std::atof(e);
  const double thr = 1e-3 * eps / (static_cast<double>(images) * static_cast<double>(ns > 0 ? ns : 1)) *
                     (grad ? 0.5 : 1.0);
  auto val = [grad](double x) {
    const pwk::K01 k = pwk::k01_of_sq(x * x);
    return grad ? k.k1_over_x * x : k.k0;
  };
  if (val(64.0) > thr) return 64.0;
  double lo = 2.0, hi = 64.0;  // val(lo) > thr >= val(hi) (K0(2) = 0.11 > any eps-scaled threshold)
  if (val(lo) <= thr) return lo;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    (val(mid) > thr ? lo : hi) = mid;
  }
  return hi;
}

long Plan::sym_items(const Opts& o, size_t n) {
  DevSys s;
  s.ns = s.nt = n;
  NearArgs a;
  const NearKind nk = near_args(s, o, DevOut{}, false, 0, 0, false, a);
  if (!near_sym_supported(nk) || n == 0) return 0;
  return near_sym_item_count(nk, n, prod_form(pz_, nk, a, n));
}

// Screened kernels (binned, masked, regime sweeps) cost very different amounts per work
// item -- c5's far tile pairs lose most images -- so their items are split by estimated
// cost (near_sym.cu near_sym_split; every rank computes the same bounds from the same
// points); the other kernels' items cost the same, split by count.
void Plan::sym_split(const DevSys& s, const Opts& o, int world, long* bounds) {
  require(world >= 1 && world <= 64, ErrorCode::Unsupported, "world size must be in [1, 64]");
  NearArgs a;
  const NearKind nk = near_args(s, o, DevOut{}, false, 0, 0, false, a);
  const long items = near_sym_supported(nk) ? near_sym_item_count(nk, s.nt, prod_form(pz_, nk, a, s.nt)) : 0;
  const bool screened = near_screened(nk, a) && s.nt >= 4096 && std::getenv("PWB_NO_BINNING") == nullptr &&
                        std::getenv("PWB_COUNT_SPLIT") == nullptr;
  if (!screened || world == 1 || items == 0) {
    for (int r = 0; r <= world; ++r) bounds[r] = items * r / world;
    return;
  }
  require(s.tgt == s.src && s.nt == s.ns, ErrorCode::Unsupported, "the symmetric near field needs the sources as targets");
  cudaStream_t st = stream_for(o);
  bin_inputs(s, a, st);  // the same sorted points sym_partial runs on
  const size_t nb = near_sym_tiles(s.nt);
  auto* rs_dev = sym_rows_.as<long long>(nb + 1);
  auto* rs_host = static_cast<long long*>(sym_rows_host_.ensure((nb + 1) * sizeof(long long)));
  const size_t bytes = near_sym_split_bytes(s.nt, items);
  void* ws = sym_split_ws_.ensure(bytes);
  long* hb = static_cast<long*>(host_checks_.ensure(65 * sizeof(long)));
  near_sym_split(nk, a, world, hb, ws, bytes, rs_dev, rs_host, st);
  for (int r = 0; r <= world; ++r) bounds[r] = hb[r];
}

int Plan::near_nout(const Opts& o) const {
  NearArgs a;
  return static_cast<int>(near_outputs(near_args(DevSys{}, o, DevOut{}, false, 0, 0, false, a)));
}

int Plan::sym_partial(const DevSys& s, const Opts& o, long begin, long end, unsigned long long* acc,
                      int* scale_exp) {
  require(s.tgt == s.src && s.nt == s.ns, ErrorCode::Unsupported,
          "the symmetric near field needs the sources as targets");
  cudaStream_t st = stream_for(o);
  NearArgs a;
  const NearKind nk = near_args(s, o, DevOut{}, false, 0, 0, false, a);
  require(near_sym_supported(nk), ErrorCode::Unsupported, "no symmetric near tile for this kernel");
  int* flag = flag_.as<int>(1);
  cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), st), "memset flag");
  a.flag = flag;
  // the fixed-point scale comes from the global strengths (every rank holds all of them,
  // so every rank scales identically and the integer reduce-scatter stays exact)
  unsigned* maxhi = fx_maxhi_.as<unsigned>(1);
  launch_fx_maxhi(a, maxhi, st);
  a.fx_maxhi = maxhi;
  const size_t nb = near_sym_tiles(s.nt);
  auto* rs_dev = sym_rows_.as<long long>(nb + 1);
  auto* rs_host = static_cast<long long*>(sym_rows_host_.ensure((nb + 1) * sizeof(long long)));
  SymRange r;
  r.begin = begin;
  r.end = end;
  r.finish = false;
  cuda_check(cudaEventRecord(ev_[2], st), "event");
  // screened kernels: the same Morton binning as the single-GPU path (every rank sorts the
  // same points identically, so the work items cover the same pairs); the tile runs into a
  // sorted-order scratch accumulator that is added back in input order, keeping the
  // accumulator layout (and the reduce-scatter slices) of the caller
  if (prod_form(pz_, nk, a, s.nt) ||
      (near_screened(nk, a) && s.nt >= 4096 && std::getenv("PWB_NO_BINNING") == nullptr)) {
    bin_inputs(s, a, st);
    const int* perm = a.out_row;
    a.out_row = nullptr;
    const int w = 3 * static_cast<int>(near_outputs(nk));
    auto* sorted = sym_fx_.as<unsigned long long>(static_cast<size_t>(w) * s.nt);
    cuda_check(cudaMemsetAsync(sorted, 0, static_cast<size_t>(w) * s.nt * sizeof(unsigned long long), st),
               "memset sorted acc");
    launch_near_sym(nk, a, st, sorted, rs_dev, rs_host, r);
    scatter_add_rows(sorted, perm, s.nt, w, acc, st);
  } else {
    launch_near_sym(nk, a, st, acc, rs_dev, rs_host, r);
  }
  cuda_check(cudaEventRecord(ev_[3], st), "event");
  near_timed_ = true;
  cuda_check(cudaGetLastError(), "near launch");
  auto* h = static_cast<unsigned*>(host_checks_.ensure(64 * sizeof(double)));
  cuda_check(cudaMemcpyAsync(h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H flag");
  cuda_check(cudaMemcpyAsync(h + 1, maxhi, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H maxhi");
  cuda_check(cudaStreamSynchronize(st), "near sync");
  if (scale_exp) *scale_exp = fx_exponent(h[1], s.ns);
  return static_cast<int>(h[0]);
}

void Plan::fixed_finish(const Opts& o, const unsigned long long* acc, size_t n, int scale_exp, const DevOut& out) {
  require(scale_exp >= -960 && scale_exp <= 960, ErrorCode::Unsupported, "fixed-point scale exponent out of range");
  NearArgs a;
  near_args(DevSys{}, o, out, false, 0, 0, false, a);
  launch_fx_finish(acc, n, a.out0, a.nout0, a.out1, a.nout1, nullptr, nullptr, 0, scale_exp, nullptr, stream_for(o));
  cuda_check(cudaGetLastError(), "fixed-point finish");
  cuda_check(cudaStreamSynchronize(stream_for(o)), "sync");
}

// Product form of the symmetric Laplace and Stokeslet tiles (near_sym_impl.cuh SymLaplace /
// SymStokes PROD): Laplace on a singly periodic cell (one image row of three) or an unskewed
// doubly periodic one with 3 x 3 images, the Stokeslet without pressure on the latter; a
// reduced precision tier (eps >= 1e-11). Host-only (the work-item count of
// pwb_near_sym_items needs no device). PWB_NO_PROD=1: off (A/B, tests).
bool prod_eligible(const periwave::Periodizer& pz, NearKind nk, size_t n) {
  const periwave::UnitCell& c = pz.cell;
  if (nk != NearKind::Laplace && nk != NearKind::Stokes) return false;
  if (nk == NearKind::Stokes && (c.periodicity != periwave::Periodicity::Doubly || pz.dlp)) return false;
  if (c.periodicity == periwave::Periodicity::Doubly && (c.xi != 0.0 || c.m0 != 1)) return false;
  if (n < 4096 || !(pz.eps >= 1e-11) || std::getenv("PWB_FULL_PRECISION") != nullptr) return false;
  if (std::getenv("PWB_NO_PROD") != nullptr || std::getenv("PWB_NO_BINNING") != nullptr) return false;
  // scaled form (d a power of two): any representable scale; unscaled form: products of up
  // to nine r^2 ~ d^18 must stay normal numbers
  int e = 0;
  if (c.d > 0.0 && std::frexp(c.d, &e) == 0.5) return e >= -400 && e <= 400;
  return c.d >= 0x1p-30 && c.d <= 0x1p30;
}
// Sets the tile's constants when eligible; the caller bins (bin_inputs scales the gathered
// points). A period that is a power of two lets the points be scaled by 2 / d exactly (the
// cheaper form, prod = 1); any other period keeps them unscaled (prod = 2).
bool prod_form(const periwave::Periodizer& pz, NearKind nk, NearArgs& a, size_t n) {
  if (!prod_eligible(pz, nk, n) || !a.lowp || a.nxi != 3) return false;
  if (a.nrow != (pz.cell.periodicity == periwave::Periodicity::Singly ? 1 : 3)) return false;
  const double d = pz.cell.d;
  int e = 0;
  if (std::frexp(d, &e) == 0.5 && std::getenv("PWB_PROD_UNSCALED") == nullptr) {
    a.prod = 1;
    a.prod_sc = std::ldexp(1.0, 2 - e);  // 2 / d
    a.prod_period = 2.0;
    const double ln2 = 0.6931471805599453094, lnsc = static_cast<double>(2 - e) * ln2;
    // Laplace: the tile's product is (sc^6 / 16) P per image row; Stokeslet: (sc^18 / 512) P
    a.prod_log_off = nk == NearKind::Laplace ? a.nrow * (4.0 * ln2 - 6.0 * lnsc) : 9.0 * ln2 - 18.0 * lnsc;
    a.prod_ln_sc2 = 2.0 * lnsc;
  } else {
    a.prod = 2;
    a.prod_sc = 1.0;
    a.prod_period = d;
    a.prod_d2 = d * d;
    a.prod_4d2 = 4.0 * (d * d);
    a.prod_log_off = 0.0;
    a.prod_ln_sc2 = 0.0;
  }
  a.prod_eta = pz.cell.eta * a.prod_sc;
  return true;
}

bool near_screened(NearKind nk, const NearArgs& a) {
  return nk == NearKind::ModHelm || nk == NearKind::ModHelmGrad || nk == NearKind::ModStokes ||
         nk == NearKind::ModStokesP || (nk == NearKind::Multipole && a.screened);
}

// Morton-ordered copies of the points and strengths; outputs keep their original
// rows through a.out_row (binning.cu explains why the screened kernels want this).
void Plan::bin_inputs(const DevSys& s, NearArgs& a, cudaStream_t st) {
  const periwave::UnitCell& c = pz_.cell;
  const double wx = c.d + std::abs(c.xi), wy = c.eta;
  BinBox box;
  box.x0 = -0.5 * wx;
  box.y0 = -0.5 * wy;
  box.inv_h = 65535.0 / std::max(wx, wy);
  const bool same = a.tgt == a.src;
  const size_t ws_bytes = morton_order_bytes(std::max(s.ns, s.nt));
  void* ws = bin_ws_.ensure(ws_bytes);
  int* ps = bin_perm_s_.as<int>(s.ns);
  morton_order(a.src, s.ns, box, ps, ws, ws_bytes, st);
  double2* src = bin_src_.as<double2>(s.ns);
  if (a.prod == 1)
    gather_scale_double2(a.src, ps, s.ns, a.prod_sc, src, st);
  else
    gather_double2(a.src, ps, s.ns, src, st);
  if (a.q) {
    double* q = bin_q_.as<double>(s.ns);
    gather_double(a.q, ps, s.ns, q, st);
    a.q = q;
  }
  if (a.vec) {
    double2* v = bin_vec_.as<double2>(s.ns);
    gather_double2(a.vec, ps, s.ns, v, st);
    a.vec = v;
  }
  if (a.nrm) {
    double2* v = bin_nrm_.as<double2>(s.ns);
    gather_double2(a.nrm, ps, s.ns, v, st);
    a.nrm = v;
  }
  if (same) {
    a.tgt = src;
    a.out_row = ps;
  } else {
    int* pt = bin_perm_t_.as<int>(s.nt);
    morton_order(a.tgt, s.nt, box, pt, ws, ws_bytes, st);
    double2* tgt = bin_tgt_.as<double2>(s.nt);
    if (a.prod == 1)
      gather_scale_double2(a.tgt, pt, s.nt, a.prod_sc, tgt, st);
    else
      gather_double2(a.tgt, pt, s.nt, tgt, st);
    a.tgt = tgt;
    a.out_row = pt;
  }
  a.src = src;
}

void Plan::near(const DevSys& s, const Opts& o, const DevOut& out, bool single, double shx, double shy,
                bool identity) {
  if (s.nt == 0 || s.ns == 0) return;
  cudaStream_t st = stream_for(o);
  NearArgs a;
  const NearKind nk = near_args(s, o, out, single, shx, shy, identity, a);
  int* flag = flag_.as<int>(1);
  // on the near branch of a captured call the tile starts at the fork: clear its flag there
  cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), branch_ ? side_[1] : st), "memset flag");
  a.flag = flag;
  const size_t nout = near_outputs(nk);
  // targets == sources (same array): every unordered pair once (near_sym.cu)
  // (below ~32K points the triangle has too few work items to fill 148 SMs; the
  // one-sided tile with source splits is faster there)
  const bool symmetric = !single && s.tgt == s.src && s.nt == s.ns && s.nt >= 32768 && near_sym_supported(nk) &&
                         std::getenv("PWB_NO_SYMMETRIC") == nullptr;
  record(2, branch_ ? side_[1] : st);  // on the branch the tile starts at the fork
  // screened kernels branch on beta*r per pair: bin so the branch is warp-uniform
  const bool screened = near_screened(nk, a);
  const NearArgs plain = a;  // unbinned, unscaled: the fp64 fallback of a product-form run
  // the product-form Laplace tile needs compact tiles (and takes its points scaled)
  const bool prod = symmetric && prod_form(pz_, nk, a, s.nt);
  if (prod || (!single && screened && s.nt >= 4096 && s.ns >= 4096 && std::getenv("PWB_NO_BINNING") == nullptr))
    bin_inputs(s, a, branch_ ? side_[1] : st);  // the tile's stream (captured calls never bin today)
  bool done = false;
  if (symmetric) {
    const size_t nb = near_sym_tiles(s.nt);
    auto* fx = sym_fx_.as<unsigned long long>(3 * s.nt * nout);
    auto* rs_dev = sym_rows_.as<long long>(nb + 1);
    auto* rs_host = static_cast<long long*>(sym_rows_host_.ensure((nb + 1) * sizeof(long long)));
    unsigned* maxhi = fx_maxhi_.as<unsigned>(1);
    launch_fx_maxhi(a, maxhi, st);
    a.fx_maxhi = maxhi;
    done = launch_near_sym(nk, a, st, fx, rs_dev, rs_host, SymRange{});
    if (prod && !done) throw_internal("product-form Laplace tile not launched");
  }
  if (!done) {
    double* ws = near_partial_.as<double>(static_cast<size_t>(kMaxSplits) * s.nt * nout);
    if (branch_) {  // a split tile runs on the near branch, its reduction here after the far pass
      a.tile_stream = side_[1];
      a.tile_done = side_done_[1];
    }
    launch_near(nk, a, st, ws, sms_);
  }
  record(3, st);
  near_timed_ = true;
  cuda_check(cudaGetLastError(), "near launch");
  // the flag lands past validate's check words (a deferred call still reads those)
  int* hflag = reinterpret_cast<int*>(static_cast<double*>(host_checks_.ensure(64 * sizeof(double))) + 56);
  cuda_check(cudaMemcpyAsync(hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H flag");
  if (defer_) {
    // deferred calls are one-sided (graph_eligible): no fixed-point fallback to run
    require(!symmetric, ErrorCode::Unsupported, "internal: symmetric tile in a deferred call");
    pending_.push_back([hflag] {
      require((*hflag & 1) == 0, ErrorCode::CoincidentSourceTarget,
              "a target coincides with a lattice image of a source");
    });
    return;
  }
  cuda_check(cudaStreamSynchronize(st), "near sync");
  require((*hflag & 1) == 0, ErrorCode::CoincidentSourceTarget, "a target coincides with a lattice image of a source");
  if (*hflag & 2) {
    // a scaled partial sum left the fixed-point range (non-finite strengths, or kernel
    // values beyond ~2^60 times the strengths): the readout was skipped; redo the near
    // field on the one-sided tile, which sums in fp64 like the reference
    cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), st), "memset flag");
    double* ws = near_partial_.as<double>(static_cast<size_t>(kMaxSplits) * s.nt * nout);
    launch_near(nk, prod ? plain : a, st, ws, sms_);
    cuda_check(cudaEventRecord(ev_[3], st), "event");
    cuda_check(cudaGetLastError(), "near launch");
    cuda_check(cudaMemcpyAsync(hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H flag");
    cuda_check(cudaStreamSynchronize(st), "near sync");
    require((*hflag & 1) == 0, ErrorCode::CoincidentSourceTarget, "a target coincides with a lattice image of a source");
  }
}

void Plan::record(int i, cudaStream_t st) {
  // inside a capture the event becomes a graph node that records on every replay
  if (defer_)
    cuda_check(cudaEventRecordWithFlags(ev_[i], st, cudaEventRecordExternal), "event");
  else
    cuda_check(cudaEventRecord(ev_[i], st), "event");
}

bool Plan::GraphKey::operator==(const GraphKey& o) const {
  return s.src == o.s.src && s.q == o.s.q && s.f == o.s.f && s.nrm == o.s.nrm && s.coef == o.s.coef &&
         s.ns == o.s.ns && s.tgt == o.s.tgt && s.nt == o.s.nt && outs == o.outs && path == o.path &&
         pressure == o.pressure && gradient == o.gradient && far == o.far && near == o.near &&
         nufft_eps == o.nufft_eps;
}

// Launch-latency-bound calls only: both passes, one-sided near tile (the symmetric tile
// needs n >= 32768 and may fall back on a status word), at most ~4M pairs.
bool Plan::graph_eligible(const DevSys& s, bool far, bool near_images) const {
  static const bool off = std::getenv("PWB_NO_GRAPH") != nullptr;
  return !off && far && near_images && s.ns > 0 && s.nt > 0 && s.nt < 32768 &&
         static_cast<double>(s.ns) * static_cast<double>(s.nt) <= 4.2e6;
}

void Plan::drop_graphs() {
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
  seen_.clear();
  no_graph_.clear();
}

bool Plan::total(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images) {
  if (graph_eligible(s, far, near_images)) return total_graphed(s, o, out, far, near_images);
  return total_eager(s, o, out, far, near_images);
}

bool Plan::total_graphed(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images) {
  // outputs: the graph writes the plan's own block (fixed pointers, so a caller that
  // allocates fresh result arrays per call still replays) and every replay copies it out
  double* const user[5] = {out.scalar, out.velocity, out.pressure, out.complex_scalar, out.gradient};
  const size_t width[5] = {1, 2, 1, 2, 2};
  GraphKey k;
  k.s = s;
  for (int i = 0; i < 5; ++i)
    if (user[i]) k.outs |= 1u << i;
  k.path = static_cast<int>(o.path);
  k.pressure = o.with_pressure;
  k.gradient = o.with_gradient;
  k.far = far;
  k.near = near_images;
  k.nufft_eps = o.nufft_eps;
  if (graph_epoch_ != buffer_epoch()) {  // a workspace moved: every captured graph is stale
    drop_graphs();
    graph_epoch_ = buffer_epoch();
  }
  cudaStream_t st = stream_for(o);
  double* own[5] = {};
  auto own_outputs = [&] {
    double* base = graph_out_.as<double>(8 * s.nt);
    size_t off = 0;
    for (int i = 0; i < 5; ++i)
      if (user[i]) {
        own[i] = base + off;
        off += width[i] * s.nt;
      }
  };
  auto launch = [&](const GraphEntry& e) {
    own_outputs();
    cuda_check(cudaGraphLaunch(e.exec, st), "graph launch");
    for (int i = 0; i < 5; ++i)
      if (user[i])
        cuda_check(cudaMemcpyAsync(user[i], own[i], width[i] * s.nt * sizeof(double), cudaMemcpyDeviceToDevice, st),
                   "graph output copy");
    count_launches(e.launches);
    cuda_check(cudaStreamSynchronize(st), "graph sync");
    far_timed_ = e.far_timed;
    near_timed_ = e.near_timed;
    for (const auto& c : e.checks) c();
    return e.accelerated;
  };
  for (const auto& e : graphs_)
    if (e.key == k) return launch(e);
  if (std::find(no_graph_.begin(), no_graph_.end(), k) != no_graph_.end())
    return total_eager(s, o, out, far, near_images);
  if (std::find(seen_.begin(), seen_.end(), k) == seen_.end()) {
    // first sighting: run eagerly (sizes every workspace and one-time setup), remember it
    own_outputs();  // size the output block now, so the capture does not move a buffer
    const bool acc = total_eager(s, o, out, far, near_images);
    if (seen_.size() >= 16) seen_.erase(seen_.begin());
    seen_.push_back(k);
    graph_epoch_ = buffer_epoch();
    return acc;
  }
  // second sighting: capture the whole call on the plan's capture stream, replay on `st`
  if (!capture_stream_) cuda_check(cudaStreamCreateWithFlags(&capture_stream_, cudaStreamNonBlocking), "stream");
  Opts oc = o;
  oc.stream = capture_stream_;
  GraphEntry e;
  e.key = k;
  const long l0 = launch_count();
  cuda_check(cudaStreamBeginCapture(capture_stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  defer_ = true;
  pending_.clear();
  cudaGraph_t graph = nullptr;
  own_outputs();
  const DevOut gout{own[0], own[1], own[2], own[3], own[4]};
  auto abandon = [&] {  // end the capture and forget it (the CUDA error state is cleared)
    defer_ = false;
    branch_ = false;
    cudaStreamEndCapture(capture_stream_, &graph);
    if (graph) cudaGraphDestroy(graph);
    graph = nullptr;
    cudaGetLastError();
    count_launches(-(launch_count() - l0));
    pending_.clear();
  };
  try {
    e.accelerated = total_eager(s, oc, gout, far, near_images);
  } catch (const CudaFailure&) {
    // the capture itself failed (an operation the driver cannot capture): this call shape
    // runs eagerly from now on
    abandon();
    no_graph_.push_back(k);
    return total_eager(s, o, out, far, near_images);
  } catch (...) {  // a host-side check of the call (argument / validation error): propagate
    abandon();
    throw;
  }
  defer_ = false;
  cudaError_t err = cudaStreamEndCapture(capture_stream_, &graph);
  if (err == cudaSuccess) err = cudaGraphInstantiate(&e.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (err != cudaSuccess) {
    cudaGetLastError();
    count_launches(-(launch_count() - l0));
    pending_.clear();
    no_graph_.push_back(k);
    return total_eager(s, o, out, far, near_images);
  }
  e.launches = launch_count() - l0;
  count_launches(-e.launches);  // captured, not run: counted on every replay instead
  e.far_timed = far_timed_;
  e.near_timed = near_timed_;
  e.checks = std::move(pending_);
  pending_.clear();
  if (graph_epoch_ != buffer_epoch()) {  // the capture itself grew a workspace: replay later
    cudaGraphExecDestroy(e.exec);
    graph_epoch_ = buffer_epoch();
    drop_graphs();
    return total_eager(s, o, out, far, near_images);
  }
  if (graphs_.size() >= 8) {
    cudaGraphExecDestroy(graphs_.front().exec);
    graphs_.erase(graphs_.begin());
  }
  graphs_.push_back(std::move(e));
  return launch(graphs_.back());
}

void Plan::ensure_side() {
  if (side_[0]) return;
  for (auto& side : side_) cuda_check(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "event");
  for (auto& e : side_done_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
}

bool Plan::total_eager(const DevSys& s, const Opts& o, const DevOut& out, bool far, bool near_images) {
  bool accelerated = false;
  cudaStream_t st = stream_for(o);
  far_timed_ = near_timed_ = false;
  // Capturing a small call (graph replay): the validation reductions and the near tile do not
  // feed the far pass (the checks are deferred to after the replay), so they become parallel
  // branches forked at the start: validation joins before the moment sum that reuses its
  // partials, the tile before the reduction of its split partials into the outputs.
  branch_ = defer_ && far && near_images;
  if (branch_) {
    ensure_side();
    cuda_check(cudaEventRecord(fork_ev_, st), "fork");
    for (auto& side : side_) cuda_check(cudaStreamWaitEvent(side, fork_ev_, 0), "fork wait");
  }
  if (far) {
    Opts ov = o;
    if (branch_) ov.stream = side_[0];
    validate(s, ov, true);
    if (branch_) cuda_check(cudaEventRecord(side_done_[0], side_[0]), "validation join");
    const periwave::ApplyPath path = resolve(o, s.ns, s.nt);
    double* coeff = coeff_ws_.as<double>(coeff_size(o, path));
    record(0, st);
    // validate just reduced these sources (on the branch: the moment sum waits for it)
    source_pass(s, o, coeff, path, true, branch_ ? side_done_[0] : nullptr);
    accelerated = target_pass(s, o, coeff, out, path);
    record(1, st);
    far_timed_ = true;
  }
  if (near_images) {
    if (!far) validate(s, o, false);
    near(s, o, out, false, 0.0, 0.0, false);
  }
  if (branch_) {  // every branch rejoins the origin stream before the capture ends
    cuda_check(cudaStreamWaitEvent(st, side_done_[0], 0), "validation join wait");
    branch_ = false;
  }
  return accelerated;
}

}  // namespace pwb
