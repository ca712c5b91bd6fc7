// The C-ABI (include/periwave_b200.h): error mapping, handles, host/device
// staging. No exception crosses this boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>

#include "engine.hpp"
#include "periwave_b200.h"

namespace pwb {
int eval_in_width(int which);
int eval_out_width(int which);
void run_eval(int which, int pde, double beta, int l, size_t n, const double* in_host, double* out_host);
double fp64_peak_probe();
int nufft_entry(int type, int backend, double eps, size_t n, const double* x, const double* c, size_t nk,
                const double* s, double* f, int memory, void* stream);
}  // namespace pwb

struct pwb_periodizer {
  periwave::Periodizer pz;
  std::mutex mu;
  std::map<int, std::unique_ptr<pwb::Plan>> plans;
  pwb::Plan& plan(int device) {
    std::lock_guard<std::mutex> g(mu);
    auto it = plans.find(device);
    if (it != plans.end()) return *it->second;
    auto p = std::make_unique<pwb::Plan>(pz, device);
    pwb::Plan& ref = *p;
    plans.emplace(device, std::move(p));
    return ref;
  }
};

namespace {

constexpr int OK = PWB_OK;
thread_local std::string g_msg;

template <class F>
int guard(F&& f) {
  try {
    g_msg.clear();
    return f();
  } catch (const periwave::Error& e) {
    g_msg = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const pwb::CudaFailure& e) {
    g_msg = e.what();
    return PWB_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    g_msg = "out of host memory";
    return PWB_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return PWB_ERR_INTERNAL;
  }
}

int fail_arg(const char* what) {
  g_msg = what;
  return PWB_ERR_INVALID_ARGUMENT;
}

periwave::UnitCell cell_from(const pwb_cell* c) {
  periwave::UnitCell u;
  u.d = c->d;
  u.xi = c->xi;
  u.eta = c->eta;
  u.periodicity = c->periodicity == PWB_SINGLY ? periwave::Periodicity::Singly : periwave::Periodicity::Doubly;
  u.m0 = c->m0;
  return u;
}

void cell_to(const periwave::UnitCell& u, pwb_cell* c) {
  c->d = u.d;
  c->xi = u.xi;
  c->eta = u.eta;
  c->periodicity = u.periodicity == periwave::Periodicity::Singly ? PWB_SINGLY : PWB_DOUBLY;
  c->m0 = u.m0;
}

int current_device(int requested) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw pwb::CudaFailure("no CUDA device available");
  }
  int dev = requested;
  if (dev < 0) pwb::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  pwb::cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  return dev;
}

pwb::Opts opts_from(const pwb_options* o) {
  pwb::Opts r;
  if (!o) return r;
  r.path = o->path == PWB_PATH_DIRECT ? periwave::ApplyPath::Direct
           : o->path == PWB_PATH_ACCELERATED ? periwave::ApplyPath::Accelerated
                                             : periwave::ApplyPath::Auto;
  r.with_pressure = o->with_pressure != 0;
  r.with_gradient = o->with_gradient != 0;
  r.nufft_eps = o->nufft_eps;
  r.stream = static_cast<cudaStream_t>(o->stream);
  return r;
}

// Stages a (possibly host-resident) system and output block on the device.
struct Staged {
  pwb::DevSys sys;
  pwb::DevOut out;
  bool host_out = false;
  double* dev_out_base = nullptr;
  size_t nt = 0;
  // host pointers to copy back into
  pwb_field* field = nullptr;
};

const double2* put(pwb::DevBuf& b, const double* h, size_t ndoubles, cudaStream_t st) {
  if (!h) return nullptr;
  double* d = b.as<double>(ndoubles);
  if (ndoubles) pwb::cuda_check(cudaMemcpyAsync(d, h, ndoubles * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
  return reinterpret_cast<const double2*>(d);
}

// Output offsets in the device output block: scalar nt, velocity 2nt, pressure nt, complex 2nt, gradient 2nt.
constexpr int kOutDoubles = 8;

void stage_in(pwb::Plan& p, const pwb_system* s, cudaStream_t st, pwb::DevSys* ds) {
  ds->ns = s->n_src;
  ds->nt = s->n_tgt;
  if (s->memory == PWB_MEM_DEVICE) {
    ds->src = reinterpret_cast<const double2*>(s->sources);
    ds->q = s->charges;
    ds->f = reinterpret_cast<const double2*>(s->forces);
    ds->nrm = reinterpret_cast<const double2*>(s->normals);
    ds->coef = reinterpret_cast<const double2*>(s->coefficients);
    ds->tgt = reinterpret_cast<const double2*>(s->targets);
    return;
  }
  ds->src = put(p.stage[0], s->sources, 2 * s->n_src, st);
  ds->q = reinterpret_cast<const double*>(put(p.stage[1], s->charges, s->n_src, st));
  ds->f = put(p.stage[2], s->forces, 2 * s->n_src, st);
  ds->nrm = put(p.stage[3], s->normals, 2 * s->n_src, st);
  ds->coef = put(p.stage[4], s->coefficients, 2 * s->n_src, st);
  // targets given as the sources array itself, or as a separate host array holding the
  // same bytes (the reference's ParticleSystem keeps two vectors, cell.hpp:58-65, so a
  // drop-in caller with targets = sources passes a copy): keep them one device array so the
  // symmetric near tile (every unordered pair once) applies. Equal bytes are equal points
  // (one O(N) memcmp, against O(N^2) pair work), so the result is the aliased call's.
  if (s->n_tgt == s->n_src && s->targets &&
      (s->targets == s->sources || std::memcmp(s->targets, s->sources, 2 * s->n_src * sizeof(double)) == 0))
    ds->tgt = ds->src;
  else
    ds->tgt = put(p.stage[5], s->targets, 2 * s->n_tgt, st);
}

// `load` copies the current host outputs in first (accumulate entry points).
void stage_out(pwb::Plan& p, pwb_field* f, size_t nt, cudaStream_t st, bool load, pwb::DevOut* out) {
  if (f->memory == PWB_MEM_DEVICE) {
    out->scalar = f->scalar;
    out->velocity = f->velocity;
    out->pressure = f->pressure;
    out->complex_scalar = f->complex_scalar;
    out->gradient = f->gradient;
    return;
  }
  double* base = p.stage[6].as<double>(kOutDoubles * nt + 8);
  double* ptrs[5] = {base, base + nt, base + 3 * nt, base + 4 * nt, base + 6 * nt};
  double* host[5] = {f->scalar, f->velocity, f->pressure, f->complex_scalar, f->gradient};
  const size_t width[5] = {1, 2, 1, 2, 2};
  for (int i = 0; i < 5; ++i)
    if (load && host[i] && nt)
      pwb::cuda_check(cudaMemcpyAsync(ptrs[i], host[i], width[i] * nt * sizeof(double), cudaMemcpyHostToDevice, st),
                      "H2D out");
  out->scalar = f->scalar ? ptrs[0] : nullptr;
  out->velocity = f->velocity ? ptrs[1] : nullptr;
  out->pressure = f->pressure ? ptrs[2] : nullptr;
  out->complex_scalar = f->complex_scalar ? ptrs[3] : nullptr;
  out->gradient = f->gradient ? ptrs[4] : nullptr;
}

void unstage_out(pwb::Plan& p, pwb_field* f, size_t nt, cudaStream_t st) {
  if (f->memory == PWB_MEM_DEVICE || nt == 0) {
    pwb::cuda_check(cudaStreamSynchronize(st), "sync");
    return;
  }
  double* base = static_cast<double*>(p.stage[6].get());
  double* ptrs[5] = {base, base + nt, base + 3 * nt, base + 4 * nt, base + 6 * nt};
  double* host[5] = {f->scalar, f->velocity, f->pressure, f->complex_scalar, f->gradient};
  const size_t width[5] = {1, 2, 1, 2, 2};
  for (int i = 0; i < 5; ++i)
    if (host[i])
      pwb::cuda_check(cudaMemcpyAsync(host[i], ptrs[i], width[i] * nt * sizeof(double), cudaMemcpyDeviceToHost, st),
                      "D2H out");
  pwb::cuda_check(cudaStreamSynchronize(st), "sync");
}

// Which outputs the apply needs, per the periodizer kind (apply.hpp:22-31).
void check_outputs(const periwave::Periodizer& pz, const pwb::Opts& o, const pwb_field* f) {
  const pwb::Kind k = pwb::kind_of(pz);
  if (k == pwb::Kind::Multipole && !f->complex_scalar) throw std::invalid_argument("complex_scalar output required");
  if (k == pwb::Kind::Velocity && !f->velocity) throw std::invalid_argument("velocity output required");
  if (k == pwb::Kind::Scalar && !f->scalar) throw std::invalid_argument("scalar output required");
  // unsupported combinations are reported by the engine's validation as Unsupported
  if (o.with_pressure && k == pwb::Kind::Velocity && !pz.dlp && !f->pressure)
    throw std::invalid_argument("pressure output required");
  if (o.with_gradient && k == pwb::Kind::Scalar && pz.pde == periwave::Pde::ModHelmholtz && !f->gradient)
    throw std::invalid_argument("gradient output required");
}

enum class Mode { Total, Far, Near, Single };

int run(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o, pwb_field* f, Mode mode, double shx = 0,
        double shy = 0, int identity = 0) {
  if (!h || !s || !f) return fail_arg("null argument");
  if ((s->n_src && !s->sources) || (s->n_tgt && !s->targets)) return fail_arg("null point array");
  return guard([&] {
    pwb_periodizer* hh = const_cast<pwb_periodizer*>(h);
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = hh->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    try {
      if (s->n_tgt > 0) check_outputs(h->pz, opt, f);  // no targets: empty result, validation still runs
    } catch (const std::invalid_argument& e) {
      return fail_arg(e.what());
    }
    cudaStream_t st = p.stream_for(opt);
    pwb::DevSys ds;
    stage_in(p, s, st, &ds);
    pwb::DevOut dout;
    const bool accumulate = mode == Mode::Near || mode == Mode::Single;
    stage_out(p, f, s->n_tgt, st, accumulate, &dout);
    bool accel = false;
    switch (mode) {
      case Mode::Total: accel = p.total(ds, opt, dout, true, true); break;
      case Mode::Far: accel = p.total(ds, opt, dout, true, false); break;
      case Mode::Near: p.total(ds, opt, dout, false, true); break;
      case Mode::Single:
        p.validate(ds, opt, false);
        p.near(ds, opt, dout, true, shx, shy, identity != 0);
        break;
    }
    unstage_out(p, f, s->n_tgt, st);
    if (mode == Mode::Total || mode == Mode::Far) f->accelerated = accel ? 1 : 0;
    return OK;
  });
}

void view_part(const periwave::ModeSet& m, pwb_part* out) {
  out->axis = m.axis == periwave::Axis::Horizontal ? PWB_AXIS_HORIZONTAL : PWB_AXIS_VERTICAL;
  out->size = m.size();
  out->phase = m.phase.data();
  out->decay_t = m.decay_t.data();
  out->decay_s = m.decay_s.data();
  out->shift_t = m.shift_t.data();
  out->shift_s = m.shift_s.data();
}

periwave::ModeSet modes_from(const pwb_part* p) {
  periwave::ModeSet m;
  m.axis = p->axis == PWB_AXIS_HORIZONTAL ? periwave::Axis::Horizontal : periwave::Axis::Vertical;
  m.phase.assign(p->phase, p->phase + p->size);
  m.decay_t.assign(p->decay_t, p->decay_t + p->size);
  m.decay_s.assign(p->decay_s, p->decay_s + p->size);
  m.shift_t.assign(p->shift_t, p->shift_t + p->size);
  m.shift_s.assign(p->shift_s, p->shift_s + p->size);
  return m;
}

std::vector<periwave::cplx> cplx_from(const double* v, size_t n) {
  std::vector<periwave::cplx> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = {v[2 * i], v[2 * i + 1]};
  return out;
}

std::vector<periwave::Mat2c> mat_from(const double* v, size_t n) {
  std::vector<periwave::Mat2c> out(n);
  for (size_t i = 0; i < n; ++i) {
    const double* e = v + 8 * i;
    out[i] = {{e[0], e[1]}, {e[2], e[3]}, {e[4], e[5]}, {e[6], e[7]}};
  }
  return out;
}

periwave::Direction dir_from(int d) {
  switch (d) {
    case PWB_NORTH: return periwave::Direction::North;
    case PWB_WEST: return periwave::Direction::West;
    case PWB_EAST: return periwave::Direction::East;
    default: return periwave::Direction::South;
  }
}

}  // namespace

namespace pwb {
pwb_periodizer* wrap_periodizer(const periwave::Periodizer& pz) {
  auto h = std::make_unique<pwb_periodizer>();
  h->pz = pz;
  return h.release();
}
}  // namespace pwb

extern "C" {

const char* pwb_last_error(void) { return g_msg.c_str(); }
const char* pwb_version(void) { return "periwave-b200 0.1 (sm_100a)"; }

int pwb_device_count(int* count) {
  if (!count) return fail_arg("null count");
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return OK;
}

int pwb_make_unit_cell(double d, double xi, double eta, int periodicity, pwb_cell* out) {
  if (!out) return fail_arg("null cell");
  return guard([&] {
    cell_to(periwave::make_unit_cell(d, xi, eta,
                                     periodicity == PWB_SINGLY ? periwave::Periodicity::Singly
                                                               : periwave::Periodicity::Doubly),
            out);
    return OK;
  });
}

int pwb_near_translations(const pwb_cell* cell, size_t cap, double* shifts, int* mn, size_t* count) {
  if (!cell || !count) return fail_arg("null argument");
  return guard([&] {
    const auto tr = periwave::near_translations(cell_from(cell));
    *count = tr.size();
    for (size_t i = 0; i < tr.size() && i < cap; ++i) {
      if (shifts) {
        shifts[2 * i] = tr[i].shift.x;
        shifts[2 * i + 1] = tr[i].shift.y;
      }
      if (mn) {
        mn[2 * i] = tr[i].m;
        mn[2 * i + 1] = tr[i].n;
      }
    }
    return OK;
  });
}

int pwb_make_periodizer(int pde, double beta, const pwb_cell* cell, double eps, pwb_periodizer** out) {
  if (!cell || !out) return fail_arg("null argument");
  if (pde < 0 || pde > 3) return fail_arg("unknown pde");
  return guard([&] {
    auto h = std::make_unique<pwb_periodizer>();
    h->pz = periwave::make_periodizer(static_cast<periwave::Pde>(pde), beta, cell_from(cell), eps);
    *out = h.release();
    return OK;
  });
}

int pwb_make_stokes_dlp_periodizer(const pwb_cell* cell, double eps, pwb_periodizer** out) {
  if (!cell || !out) return fail_arg("null argument");
  return guard([&] {
    auto h = std::make_unique<pwb_periodizer>();
    h->pz = periwave::make_stokes_dlp_periodizer(cell_from(cell), eps);
    *out = h.release();
    return OK;
  });
}

int pwb_make_multipole_periodizer(int pde, double beta, int l, const pwb_cell* cell, double eps,
                                  pwb_periodizer** out) {
  if (!cell || !out) return fail_arg("null argument");
  if (pde < 0 || pde > 3) return fail_arg("unknown pde");
  return guard([&] {
    auto h = std::make_unique<pwb_periodizer>();
    h->pz = periwave::make_multipole_periodizer(static_cast<periwave::Pde>(pde), beta, l, cell_from(cell), eps);
    *out = h.release();
    return OK;
  });
}

void pwb_periodizer_free(pwb_periodizer* pz) { delete pz; }

size_t pwb_periodizer_rank(const pwb_periodizer* pz) { return pz ? pz->pz.rank() : 0; }

int pwb_truncation_order(const pwb_cell* cell, double eps, int* out) {
  if (!cell || !out) return fail_arg("null argument");
  return guard([&] {
    *out = periwave::truncation_order(cell_from(cell), eps);
    return OK;
  });
}

int pwb_periodizer_get_info(const pwb_periodizer* h, pwb_periodizer_info* out) {
  if (!h || !out) return fail_arg("null argument");
  const periwave::Periodizer& pz = h->pz;
  out->pde = static_cast<int>(pz.pde);
  out->beta = pz.beta;
  cell_to(pz.cell, &out->cell);
  out->eps = pz.eps;
  out->dlp = pz.dlp ? 1 : 0;
  out->multipole_order = pz.multipole_order;
  out->requires_neutrality = pz.requires_neutrality ? 1 : 0;
  out->n_parts[PWB_PART_SCALAR] = static_cast<int>(pz.scalar_parts.size());
  out->n_parts[PWB_PART_BLOCK] = static_cast<int>(pz.block_parts.size());
  out->n_parts[PWB_PART_PRESSURE] = static_cast<int>(pz.pressure_parts.size());
  out->n_parts[PWB_PART_STRESSLET] = static_cast<int>(pz.stresslet_parts.size());
  return OK;
}

int pwb_periodizer_get_part(const pwb_periodizer* h, int kind, int index, pwb_part* out) {
  if (!h || !out) return fail_arg("null argument");
  const periwave::Periodizer& pz = h->pz;
  std::memset(out, 0, sizeof *out);
  out->kind = kind;
  auto bad = [&] { return fail_arg("part index out of range"); };
  switch (kind) {
    case PWB_PART_SCALAR: {
      if (index < 0 || index >= static_cast<int>(pz.scalar_parts.size())) return bad();
      const auto& p = pz.scalar_parts[index];
      view_part(p.modes, out);
      out->dir = static_cast<int>(p.dir);
      out->flag = p.take_real ? 1 : 0;
      out->has_m0 = p.has_m0;
      out->t[0] = reinterpret_cast<const double*>(p.diag.data());
      out->m0[0] = p.m0_coef;
      return OK;
    }
    case PWB_PART_BLOCK: {
      if (index < 0 || index >= static_cast<int>(pz.block_parts.size())) return bad();
      const auto& p = pz.block_parts[index];
      view_part(p.modes, out);
      out->dir = static_cast<int>(p.dir);
      out->flag = (p.take_real ? 1 : 0) | (p.three_term ? 2 : 0);
      out->has_m0 = p.has_m0;
      out->t[0] = reinterpret_cast<const double*>(p.diag_a.data());
      out->t[1] = reinterpret_cast<const double*>(p.diag_b.data());
      out->m0[0] = p.m0_mat.a11;
      out->m0[1] = p.m0_mat.a12;
      out->m0[2] = p.m0_mat.a21;
      out->m0[3] = p.m0_mat.a22;
      return OK;
    }
    case PWB_PART_PRESSURE: {
      if (index < 0 || index >= static_cast<int>(pz.pressure_parts.size())) return bad();
      const auto& p = pz.pressure_parts[index];
      view_part(p.modes, out);
      out->dir = static_cast<int>(p.dir);
      out->has_m0 = p.has_m0;
      out->t[0] = reinterpret_cast<const double*>(p.diag.data());
      out->t[1] = reinterpret_cast<const double*>(p.row.data());
      out->m0[0] = p.m0_coef;
      out->m0[1] = p.m0_row.x;
      out->m0[2] = p.m0_row.y;
      return OK;
    }
    case PWB_PART_STRESSLET: {
      if (index < 0 || index >= static_cast<int>(pz.stresslet_parts.size())) return bad();
      const auto& p = pz.stresslet_parts[index];
      view_part(p.modes, out);
      out->dir = static_cast<int>(p.dir);
      out->has_m0 = p.has_m0;
      out->t[0] = reinterpret_cast<const double*>(p.a1.data());
      out->t[1] = reinterpret_cast<const double*>(p.a2.data());
      out->t[2] = reinterpret_cast<const double*>(p.smat.data());
      out->t[3] = reinterpret_cast<const double*>(p.sa.data());
      out->t[4] = reinterpret_cast<const double*>(p.sb.data());
      out->t[5] = reinterpret_cast<const double*>(p.off.data());
      out->m0[0] = p.m0_coef;
      return OK;
    }
    default:
      return fail_arg("unknown part kind");
  }
}

int pwb_periodizer_new(int pde, double beta, const pwb_cell* cell, double eps, int dlp, int multipole_order,
                       int requires_neutrality, pwb_periodizer** out) {
  if (!cell || !out) return fail_arg("null argument");
  if (pde < 0 || pde > 3) return fail_arg("unknown pde");
  return guard([&] {
    auto h = std::make_unique<pwb_periodizer>();
    h->pz.pde = static_cast<periwave::Pde>(pde);
    h->pz.beta = beta;
    h->pz.cell = cell_from(cell);
    h->pz.eps = eps;
    h->pz.dlp = dlp != 0;
    h->pz.multipole_order = multipole_order;
    h->pz.requires_neutrality = requires_neutrality != 0;
    *out = h.release();
    return OK;
  });
}

int pwb_periodizer_add_part(pwb_periodizer* h, const pwb_part* p) {
  if (!h || !p) return fail_arg("null argument");
  if (p->size && (!p->phase || !p->decay_t || !p->decay_s || !p->shift_t || !p->shift_s || !p->t[0]))
    return fail_arg("null table");
  return guard([&] {
    std::lock_guard<std::mutex> g(h->mu);
    h->plans.clear();  // tables changed: device plans are rebuilt lazily
    const size_t n = p->size;
    switch (p->kind) {
      case PWB_PART_SCALAR: {
        periwave::ScalarPart s;
        s.dir = dir_from(p->dir);
        s.modes = modes_from(p);
        s.diag = cplx_from(p->t[0], n);
        s.take_real = (p->flag & 1) != 0;
        s.has_m0 = p->has_m0 != 0;
        s.m0_coef = p->m0[0];
        h->pz.scalar_parts.push_back(std::move(s));
        break;
      }
      case PWB_PART_BLOCK: {
        periwave::BlockPart b;
        b.dir = dir_from(p->dir);
        b.modes = modes_from(p);
        b.diag_a = mat_from(p->t[0], n);
        if (p->t[1]) b.diag_b = mat_from(p->t[1], n);
        b.take_real = (p->flag & 1) != 0;
        b.three_term = (p->flag & 2) != 0;
        b.has_m0 = p->has_m0 != 0;
        b.m0_mat = {p->m0[0], p->m0[1], p->m0[2], p->m0[3]};
        h->pz.block_parts.push_back(std::move(b));
        break;
      }
      case PWB_PART_PRESSURE: {
        periwave::PressurePart q;
        q.dir = dir_from(p->dir);
        q.modes = modes_from(p);
        q.diag = cplx_from(p->t[0], n);
        const auto rows = cplx_from(p->t[1], 2 * n);
        for (size_t r = 0; r < n; ++r) q.row.push_back({rows[2 * r], rows[2 * r + 1]});
        q.has_m0 = p->has_m0 != 0;
        q.m0_coef = p->m0[0];
        q.m0_row = {p->m0[1], p->m0[2]};
        h->pz.pressure_parts.push_back(std::move(q));
        break;
      }
      case PWB_PART_STRESSLET: {
        periwave::StressletPart q;
        q.dir = dir_from(p->dir);
        q.modes = modes_from(p);
        q.a1 = mat_from(p->t[0], n);
        q.a2 = mat_from(p->t[1], n);
        q.smat = mat_from(p->t[2], n);
        q.sa = cplx_from(p->t[3], n);
        q.sb = cplx_from(p->t[4], n);
        q.off = cplx_from(p->t[5], n);
        q.has_m0 = p->has_m0 != 0;
        q.m0_coef = p->m0[0];
        h->pz.stresslet_parts.push_back(std::move(q));
        break;
      }
      default:
        return fail_arg("unknown part kind");
    }
    return OK;
  });
}

void pwb_options_default(pwb_options* o) {
  if (!o) return;
  o->path = PWB_PATH_AUTO;
  o->threads = 1;
  o->with_pressure = 0;
  o->nufft_eps = 0.0;
  o->with_gradient = 0;
  o->device = -1;
  o->stream = nullptr;
}

int pwb_total_field(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out) {
  return run(pz, sys, opt, out, Mode::Total);
}

int pwb_apply_far(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out) {
  return run(pz, sys, opt, out, Mode::Far);
}

int pwb_accumulate(const pwb_periodizer* pz, const pwb_system* sys, double shift_x, double shift_y,
                   int identity_shift, const pwb_options* opt, pwb_field* out) {
  return run(pz, sys, opt, out, Mode::Single, shift_x, shift_y, identity_shift);
}

int pwb_near_field(const pwb_periodizer* pz, const pwb_system* sys, const pwb_options* opt, pwb_field* out) {
  return run(pz, sys, opt, out, Mode::Near);
}

int pwb_choose_path(const pwb_periodizer* pz, size_t n_src, size_t n_tgt, int* path) {
  if (!pz || !path) return fail_arg("null argument");
  return guard([&] {
    *path = static_cast<int>(periwave::choose_path(pz->pz, n_src, n_tgt));
    return OK;
  });
}

int pwb_far_coeff_size(const pwb_periodizer* h, const pwb_options* o, size_t ns_total, size_t nt_total, size_t* n) {
  if (!h || !n) return fail_arg("null argument");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    const pwb::Opts opt = opts_from(o);
    *n = p.coeff_size(opt, p.resolve(opt, ns_total, nt_total));
    return OK;
  });
}

// The path of a sharded apply is resolved from the global counts (choose_path,
// apply.cpp:409-415); 0 means "this shard is the whole problem".
int pwb_far_source_pass(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o, size_t ns_total,
                        size_t nt_total, double* coeff) {
  if (!h || !s || !coeff) return fail_arg("null argument");
  if (s->memory != PWB_MEM_DEVICE) return fail_arg("sharded passes take device memory");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevSys ds;
    stage_in(p, s, p.stream_for(opt), &ds);
    const size_t nt_local = ds.nt;
    ds.nt = 0;
    p.validate(ds, opt, true, /*neutrality=*/false);  // neutrality is a property of the global system
    const auto path = p.resolve(opt, ns_total ? ns_total : s->n_src, nt_total ? nt_total : nt_local);
    p.source_pass(ds, opt, coeff, path);
    pwb::cuda_check(cudaStreamSynchronize(p.stream_for(opt)), "sync");
    return OK;
  });
}

int pwb_far_target_pass(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o, size_t ns_total,
                        size_t nt_total, const double* coeff, pwb_field* f) {
  if (!h || !s || !coeff || !f) return fail_arg("null argument");
  if (s->memory != PWB_MEM_DEVICE || f->memory != PWB_MEM_DEVICE) return fail_arg("sharded passes take device memory");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevSys ds;
    stage_in(p, s, p.stream_for(opt), &ds);
    pwb::DevOut dout;
    stage_out(p, f, s->n_tgt, p.stream_for(opt), false, &dout);
    const auto path = p.resolve(opt, ns_total ? ns_total : s->n_src, nt_total ? nt_total : s->n_tgt);
    f->accelerated = p.target_pass(ds, opt, coeff, dout, path) ? 1 : 0;
    pwb::cuda_check(cudaStreamSynchronize(p.stream_for(opt)), "sync");
    return OK;
  });
}

namespace {
periwave::ParticleSystem host_system(const pwb_system* s) {
  auto v2 = [](const double* p, size_t n) {
    std::vector<periwave::Vec2> v(p ? n : 0);
    for (size_t i = 0; i < v.size(); ++i) v[i] = {p[2 * i], p[2 * i + 1]};
    return v;
  };
  periwave::ParticleSystem ps;
  ps.sources = v2(s->sources, s->n_src);
  if (s->charges) ps.charges.assign(s->charges, s->charges + s->n_src);
  ps.forces = v2(s->forces, s->n_src);
  ps.normals = v2(s->normals, s->n_src);
  if (s->coefficients)
    for (size_t i = 0; i < s->n_src; ++i) ps.coefficients.emplace_back(s->coefficients[2 * i], s->coefficients[2 * i + 1]);
  ps.targets = v2(s->targets, s->n_tgt);
  return ps;
}

periwave::ApplyOptions api_options(const pwb_options* o) {
  periwave::ApplyOptions a;
  if (!o) return a;
  a.path = o->path == PWB_PATH_DIRECT ? periwave::ApplyPath::Direct
           : o->path == PWB_PATH_ACCELERATED ? periwave::ApplyPath::Accelerated
                                             : periwave::ApplyPath::Auto;
  a.threads = o->threads;
  a.with_pressure = o->with_pressure != 0;
  a.nufft_eps = o->nufft_eps;
  a.with_gradient = o->with_gradient != 0;
  a.device = o->device;
  a.stream = o->stream;
  return a;
}
}  // namespace

int pwb_brute_force_far(const pwb_periodizer* h, const pwb_system* s, int shells, const pwb_options* o,
                        pwb_field* f) {
  if (!h || !s || !f) return fail_arg("null argument");
  if (s->memory != PWB_MEM_HOST || f->memory != PWB_MEM_HOST) return fail_arg("validation tools take host memory");
  return guard([&] {
    const periwave::FieldResult r = periwave::brute_force_far(h->pz, host_system(s), shells, api_options(o));
    const size_t nt = s->n_tgt;
    if (f->scalar && r.scalar.size() == nt) std::copy(r.scalar.begin(), r.scalar.end(), f->scalar);
    if (f->velocity && r.velocity.size() == nt)
      for (size_t i = 0; i < nt; ++i) {
        f->velocity[2 * i] = r.velocity[i].x;
        f->velocity[2 * i + 1] = r.velocity[i].y;
      }
    if (f->complex_scalar && r.complex_scalar.size() == nt)
      for (size_t i = 0; i < nt; ++i) {
        f->complex_scalar[2 * i] = r.complex_scalar[i].real();
        f->complex_scalar[2 * i + 1] = r.complex_scalar[i].imag();
      }
    return OK;
  });
}

int pwb_periodicity_residual(const pwb_periodizer* h, const pwb_system* s, int samples, const pwb_options* o,
                             double* e1, double* e2, double* scale) {
  if (!h || !s || !e1 || !e2 || !scale) return fail_arg("null argument");
  if (s->memory != PWB_MEM_HOST) return fail_arg("validation tools take host memory");
  return guard([&] {
    const periwave::ResidualReport r = periwave::periodicity_residual(h->pz, host_system(s), samples, api_options(o));
    *e1 = r.e1;
    *e2 = r.e2;
    *scale = r.scale;
    return OK;
  });
}

int pwb_near_sym_items(const pwb_periodizer* h, size_t n, const pwb_options* o, long* n_items, int* nout) {
  if (!h || !n_items) return fail_arg("null argument");
  return guard([&] {
    const pwb::Opts opt = opts_from(o);
    const pwb::NearKind k = pwb::near_kind_of(h->pz, opt.with_pressure, opt.with_gradient);
    // the tile variant decides the work-item shape (host-only: no device needed to count)
    *n_items = pwb::near_sym_supported(k) ? pwb::near_sym_item_count(k, n, pwb::prod_eligible(h->pz, k, n)) : 0;
    if (nout) *nout = static_cast<int>(pwb::near_outputs(k));
    return OK;
  });
}

int pwb_near_sym_partial(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o, long item_begin,
                         long item_end, int64_t* acc, int* scale_exp, int* status) {
  if (!h || !s || !acc || !scale_exp || !status) return fail_arg("null argument");
  if (s->memory != PWB_MEM_DEVICE) return fail_arg("sharded passes take device memory");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevSys ds;
    stage_in(p, s, p.stream_for(opt), &ds);
    p.validate(ds, opt, false, /*neutrality=*/true);
    *status = p.sym_partial(ds, opt, item_begin, item_end, reinterpret_cast<unsigned long long*>(acc), scale_exp);
    return OK;
  });
}

int pwb_near_sym_split(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o, int world,
                       long* bounds) {
  if (!h || !s || !bounds) return fail_arg("null argument");
  if (s->memory != PWB_MEM_DEVICE) return fail_arg("sharded passes take device memory");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevSys ds;
    stage_in(p, s, p.stream_for(opt), &ds);
    p.sym_split(ds, opt, world, bounds);
    return OK;
  });
}

int pwb_fixed_to_field(const pwb_periodizer* h, const pwb_options* o, const int64_t* acc, size_t n, int scale_exp,
                       pwb_field* f) {
  if (!h || !acc || !f) return fail_arg("null argument");
  if (f->memory != PWB_MEM_DEVICE) return fail_arg("fixed-point conversion takes device memory");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevOut dout;
    stage_out(p, f, n, p.stream_for(opt), false, &dout);
    p.fixed_finish(opt, reinterpret_cast<const unsigned long long*>(acc), n, scale_exp, dout);
    return OK;
  });
}

int pwb_validate(const pwb_periodizer* h, const pwb_system* s, const pwb_options* o) {
  if (!h || !s) return fail_arg("null argument");
  return guard([&] {
    const int dev = current_device(o ? o->device : -1);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    pwb::Opts opt = opts_from(o);
    pwb::DevSys ds;
    stage_in(p, s, p.stream_for(opt), &ds);
    p.validate(ds, opt, true);
    return OK;
  });
}

int pwb_nufft_type1(int backend, double eps, size_t n, const double* x, const double* c, size_t nmodes, double* f,
                    int memory, void* stream) {
  return guard([&] { return pwb::nufft_entry(1, backend, eps, n, x, c, nmodes, nullptr, f, memory, stream); });
}

int pwb_nufft_type2(int backend, double eps, size_t n, const double* x, size_t nmodes, const double* f, double* c,
                    int memory, void* stream) {
  return guard([&] { return pwb::nufft_entry(2, backend, eps, n, x, f, nmodes, nullptr, c, memory, stream); });
}

int pwb_nufft_type3(int backend, double eps, size_t n, const double* x, const double* c, size_t nk, const double* s,
                    double* f, int memory, void* stream) {
  return guard([&] { return pwb::nufft_entry(3, backend, eps, n, x, c, nk, s, f, memory, stream); });
}

int pwb_fast_nufft_available(void) { return 1; }

int pwb_eval_kernel(int which, int pde, double beta, int l, size_t n, const double* in, double* out) {
  if (which < 0 || which > 12) return fail_arg("unknown kernel");
  if (n && (!in || !out)) return fail_arg("null argument");
  return guard([&] {
    current_device(-1);
    if (n) pwb::run_eval(which, pde, beta, l, n, in, out);
    return OK;
  });
}

int pwb_launch_count(long* count) {
  if (!count) return fail_arg("null count");
  *count = pwb::launch_count();
  return OK;
}

int pwb_last_phase_ms(const pwb_periodizer* h, int device, double* far_ms, double* near_ms) {
  if (!h || !far_ms || !near_ms) return fail_arg("null argument");
  return guard([&] {
    const int dev = current_device(device);
    pwb::Plan& p = const_cast<pwb_periodizer*>(h)->plan(dev);
    std::lock_guard<std::mutex> lock(p.mutex());
    p.phase_ms(far_ms, near_ms);
    return OK;
  });
}

int pwb_fp64_peak_probe(int device, double* tflops) {
  if (!tflops) return fail_arg("null argument");
  return guard([&] {
    current_device(device);
    *tflops = pwb::fp64_peak_probe();
    return OK;
  });
}

int pwb_rng_uniform(uint64_t seed, size_t n, double* out) {
  if (n && !out) return fail_arg("null argument");
  periwave::Rng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.uniform();
  return OK;
}

}  // extern "C"
