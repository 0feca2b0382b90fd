// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A thin extern "C" driver around the *unmodified* reference library
// (cardwave, /root/reference/proj/core), compiled by oracle/Makefile into
// oracle/_ref/libcwref.so. Python tests (tests/) and bench.py's reference /
// cpu_baseline legs load it with ctypes to obtain the reference's own answers
// on the same inputs as the GPU path:
//   * problem setup: build_regular_sheet + assign_fibrosis + build_diffusion_field
//     + assemble (mesh.cpp:72-122, fem.cpp:21-192)
//   * cell models: make_model + CellModel::rates (ionic.cpp:59, ionic.hpp:33)
//   * the hot path: diffusion_substep (fem.cpp:194-207), StrangIntegrator::advance
//     (splitting.cpp:171-181), run_simulation (splitting.cpp:219-294)
//   * the adaptation rules: reaction_substeps / diffusion_substeps / k_max_for
//     (splitting.cpp:48-72)
//   * diastolic_threshold (stimulus.cpp:115-157)
// Nothing here re-implements reference logic; it only marshals plain arrays.
#include "cardwave/errors.hpp"
#include "cardwave/fem.hpp"
#include "cardwave/ionic.hpp"
#include "cardwave/mesh.hpp"
#include "cardwave/output.hpp"
#include "cardwave/postprocess.hpp"
#include "cardwave/splitting.hpp"
#include "cardwave/stimulus.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

using namespace cardwave;

namespace {

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
}

// Status codes shared with include/cwgpu.h.
constexpr int kOk = 0, kValidation = 2, kInstability = 3, kIo = 4, kOther = 9;

}  // namespace

struct cwref_problem {
  Mesh mesh;
  DiffusionField field;
  AssembledOperator op;
  std::vector<std::shared_ptr<const CellModel>> models;
  std::vector<int> model_of_tag;
  Protocol protocol;
  std::unique_ptr<ProtocolIndex> index;
  SimulationSetup setup;
  SchemeConfig cfg;
  std::unique_ptr<StrangIntegrator> integrator;
  NodeStateArray state;
  SimulationResult result;
  long err_node = -1;
  double err_t = 0.0;
};

extern "C" {

// ---------------------------------------------------------------- setup
cwref_problem* cwref_sheet(double lx, double ly, double h, double angle_rad, double d0_myo,
                           double d0_fib, double rho, double fib_fraction, std::uint64_t seed,
                           char* err, int errlen) {
  try {
    auto p = std::make_unique<cwref_problem>();
    p->mesh = build_regular_sheet(lx, ly, h, angle_rad);
    if (fib_fraction > 0.0) p->mesh = assign_fibrosis(p->mesh, fib_fraction, seed);
    p->field = build_diffusion_field(p->mesh, d0_myo, d0_fib, rho);
    p->op = assemble(p->mesh, p->field);
    return p.release();
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void cwref_free(cwref_problem* p) { delete p; }

std::int64_t cwref_n(const cwref_problem* p) { return p->op.rows(); }
std::int64_t cwref_nnz(const cwref_problem* p) { return static_cast<std::int64_t>(p->op.val.size()); }
double cwref_dt_s(const cwref_problem* p) { return p->op.dt_s; }
int cwref_n_tags(const cwref_problem* p) { return static_cast<int>(p->mesh.tag_names.size()); }

void cwref_csr(const cwref_problem* p, std::int64_t* row_ptr, std::int64_t* col, double* val,
               double* mass) {
  std::memcpy(row_ptr, p->op.row_ptr.data(), p->op.row_ptr.size() * sizeof(std::int64_t));
  std::memcpy(col, p->op.col.data(), p->op.col.size() * sizeof(std::int64_t));
  std::memcpy(val, p->op.val.data(), p->op.val.size() * sizeof(double));
  std::memcpy(mass, p->op.lumped_mass.data(), p->op.lumped_mass.size() * sizeof(double));
}

void cwref_node_tags(const cwref_problem* p, std::int32_t* tags_out) {
  std::memcpy(tags_out, p->mesh.node_tags.data(), p->mesh.node_tags.size() * sizeof(std::int32_t));
}

// tag name of id t into buf
void cwref_tag_name(const cwref_problem* p, int t, char* buf, int len) {
  set_err(buf, len, p->mesh.tag_names[static_cast<std::size_t>(t)]);
}

// RegionSelector kinds in declaration order (mesh.hpp:50-58):
// 0 x_le, 1 x_ge, 2 y_le, 3 y_ge, 4 rectangle, 5 node_set, 6 disc.
// prm = {value, x0, x1, y0, y1, cx, cy, radius}
std::int64_t cwref_select(const cwref_problem* p, int kind, const double* prm,
                          const std::int64_t* set_nodes, std::int64_t n_set, std::int64_t* out,
                          std::int64_t cap) {
  RegionSelector sel;
  sel.kind = static_cast<RegionSelector::Kind>(kind);
  sel.value = prm[0];
  sel.x0 = prm[1];
  sel.x1 = prm[2];
  sel.y0 = prm[3];
  sel.y1 = prm[4];
  sel.cx = prm[5];
  sel.cy = prm[6];
  sel.radius = prm[7];
  for (std::int64_t i = 0; i < n_set; ++i) sel.nodes.push_back(set_nodes[i]);
  const auto nodes = select_nodes(p->mesh, sel);
  const std::int64_t m = static_cast<std::int64_t>(nodes.size());
  for (std::int64_t i = 0; i < m && i < cap; ++i) out[i] = nodes[static_cast<std::size_t>(i)];
  return m;
}

std::int64_t cwref_nearest(const cwref_problem* p, double x, double y) {
  return p->mesh.nearest_node(x, y);
}

// Wire models: names[t] is the model for tag id t (all tags must be covered).
int cwref_set_models(cwref_problem* p, const char* const* names, int n_names, char* err,
                     int errlen) {
  try {
    p->models.clear();
    p->model_of_tag.assign(p->mesh.tag_names.size(), -1);
    std::vector<std::string> seen;
    for (int t = 0; t < n_names && t < static_cast<int>(p->mesh.tag_names.size()); ++t) {
      int mid = -1;
      for (std::size_t q = 0; q < seen.size(); ++q)
        if (seen[q] == names[t]) mid = static_cast<int>(q);
      if (mid < 0) {
        p->models.push_back(make_model(names[t]));
        seen.push_back(names[t]);
        mid = static_cast<int>(seen.size() - 1);
      }
      p->model_of_tag[static_cast<std::size_t>(t)] = mid;
    }
    return kOk;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return kValidation;
  }
}

// Append a stimulus: node list (already selected), timing, optional period (NaN = none).
int cwref_add_stimulus(cwref_problem* p, const std::int64_t* nodes, std::int64_t n, double t0,
                       double dur, double amp, double period) {
  Stimulus s;
  s.nodes.assign(nodes, nodes + n);
  s.t_start_ms = t0;
  s.duration_ms = dur;
  s.amplitude = amp;
  if (!std::isnan(period)) s.period_ms = period;
  p->protocol.entries.push_back(std::move(s));
  return kOk;
}

void cwref_clear_stimuli(cwref_problem* p) { p->protocol.entries.clear(); }

int cwref_state_stride(const cwref_problem* p) {
  int stride = 1;
  for (const auto& m : p->models) stride = std::max(stride, m->state_count());
  return stride;
}

// Initial state from model rest states (make_initial_state, splitting.cpp:183).
int cwref_init_state(cwref_problem* p, char* err, int errlen) {
  try {
    p->state = make_initial_state(p->mesh, p->models, p->model_of_tag);
    return kOk;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return kValidation;
  }
}

void cwref_get_state(const cwref_problem* p, double* v, double* s, double* last_dvdt,
                     std::uint8_t* model_of_node) {
  const auto& st = p->state;
  if (v) std::memcpy(v, st.v.data(), st.v.size() * sizeof(double));
  if (s) std::memcpy(s, st.s.data(), st.s.size() * sizeof(double));
  if (last_dvdt) std::memcpy(last_dvdt, st.last_dvdt.data(), st.last_dvdt.size() * sizeof(double));
  if (model_of_node) std::memcpy(model_of_node, st.model_of_node.data(), st.model_of_node.size());
}

void cwref_put_state(cwref_problem* p, const double* v, const double* s, const double* last_dvdt) {
  auto& st = p->state;
  if (v) std::memcpy(st.v.data(), v, st.v.size() * sizeof(double));
  if (s) std::memcpy(st.s.data(), s, st.s.size() * sizeof(double));
  if (last_dvdt) std::memcpy(st.last_dvdt.data(), last_dvdt, st.last_dvdt.size() * sizeof(double));
}

// ---------------------------------------------------------------- hot path
void cwref_diffusion_substep(const cwref_problem* p, const double* v, double dt_sub, double* out) {
  std::vector<double> vin(v, v + p->op.rows()), vout;
  diffusion_substep(p->op, vin, dt_sub, vout);
  std::memcpy(out, vout.data(), vout.size() * sizeof(double));
}

static void fill_cfg(SchemeConfig& c, int scheme, double dt, double t_end, int k0_up, int k0_down,
                     int strict, double record_interval, int workers) {
  c.scheme = static_cast<Scheme>(scheme);
  c.dt_ms = dt;
  c.t_end_ms = t_end;
  c.k0_up = k0_up;
  c.k0_down = k0_down;
  c.strict_substeps = strict != 0;
  c.record_interval_ms = record_interval;
  c.workers = workers;
}

static void build_setup(cwref_problem* p, const std::int64_t* probes, int n_probes, double lat_thr) {
  p->index = std::make_unique<ProtocolIndex>(p->protocol, p->mesh.node_count());
  p->setup = SimulationSetup{};
  p->setup.op = &p->op;
  p->setup.models = p->models;
  p->setup.protocol = p->index.get();
  p->setup.lat_threshold_mv = lat_thr;
  for (int i = 0; i < n_probes; ++i) {
    Probe pr;
    pr.node = probes[i];
    pr.name = "p" + std::to_string(i);
    p->setup.probes.push_back(pr);
  }
}

// StrangIntegrator construction for step-wise driving (advance()).
int cwref_integrator(cwref_problem* p, int scheme, double dt, double t_end, int k0_up, int k0_down,
                     int strict, int workers, char* err, int errlen) {
  try {
    fill_cfg(p->cfg, scheme, dt, t_end, k0_up, k0_down, strict, 1.0, workers);
    build_setup(p, nullptr, 0, 0.0);
    p->integrator = std::make_unique<StrangIntegrator>(p->setup, p->cfg);
    return kOk;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return kValidation;
  }
}

int cwref_advance(cwref_problem* p, double t, std::int64_t step, std::int64_t n_steps,
                  std::int64_t* bad_node, double* bad_t, char* err, int errlen) {
  try {
    p->integrator->advance(p->state, t, step, n_steps);
    return kOk;
  } catch (const InstabilityError& e) {
    if (bad_node) *bad_node = e.node_index;
    if (bad_t) *bad_t = e.time_ms;
    set_err(err, errlen, e.what());
    return kInstability;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return kValidation;
  }
}

void cwref_integrator_info(const cwref_problem* p, double* dt_eff, int* l, double* dt_ad,
                           int* k_max_global, double* timing3) {
  *dt_eff = p->integrator->dt_effective();
  *l = p->integrator->plan().l;
  *dt_ad = p->integrator->plan().dt_ad;
  *k_max_global = p->integrator->k_max_global();
  if (timing3) {
    timing3[0] = p->integrator->timing().reaction_ms;
    timing3[1] = p->integrator->timing().diffusion_ms;
    timing3[2] = p->integrator->timing().total_ms;
  }
}

void cwref_integrator_khist(const cwref_problem* p, std::int64_t* out) {
  const auto& h = p->integrator->k_histogram();
  for (std::size_t i = 0; i < h.size(); ++i) out[i] = h[i];
}

// Full run_simulation from the current state (moved in; result kept).
int cwref_run(cwref_problem* p, int scheme, double dt, double t_end, int k0_up, int k0_down,
              int strict, double record_interval, int workers, const std::int64_t* probes,
              int n_probes, double lat_threshold, char* err, int errlen) {
  try {
    fill_cfg(p->cfg, scheme, dt, t_end, k0_up, k0_down, strict, record_interval, workers);
    build_setup(p, probes, n_probes, lat_threshold);
    p->result = run_simulation(p->state, p->setup, p->cfg);
    p->state = p->result.final_state;
    p->err_node = -1;
    return kOk;
  } catch (const InstabilityError& e) {
    p->err_node = e.node_index;
    p->err_t = e.time_ms;
    set_err(err, errlen, e.what());
    return kInstability;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return kValidation;
  }
}

void cwref_run_error(const cwref_problem* p, std::int64_t* node, double* t) {
  *node = p->err_node;
  *t = p->err_t;
}

// result getters
std::int64_t cwref_res_n_steps(const cwref_problem* p) { return p->result.n_steps; }
int cwref_res_khist_len(const cwref_problem* p) {
  return static_cast<int>(p->result.k_histogram.size());
}
void cwref_res_khist(const cwref_problem* p, std::int64_t* out) {
  for (std::size_t i = 0; i < p->result.k_histogram.size(); ++i) out[i] = p->result.k_histogram[i];
}
void cwref_res_plan(const cwref_problem* p, double* dt_eff, double* dt_s, int* l, double* dt_ad) {
  *dt_eff = p->result.dt_effective;
  *dt_s = p->result.dt_s;
  *l = p->result.plan.l;
  *dt_ad = p->result.plan.dt_ad;
}
void cwref_res_timing(const cwref_problem* p, double* t4) {
  t4[0] = p->result.timing.total_ms;
  t4[1] = p->result.timing.reaction_ms;
  t4[2] = p->result.timing.diffusion_ms;
  t4[3] = p->result.timing.recording_ms;
}
std::int64_t cwref_res_n_samples(const cwref_problem* p) {
  return p->result.traces.empty() ? 0 : static_cast<std::int64_t>(p->result.traces[0].t_ms.size());
}
void cwref_res_trace(const cwref_problem* p, int probe, double* t, double* v) {
  const auto& tr = p->result.traces[static_cast<std::size_t>(probe)];
  std::memcpy(t, tr.t_ms.data(), tr.t_ms.size() * sizeof(double));
  std::memcpy(v, tr.v_mv.data(), tr.v_mv.size() * sizeof(double));
}
void cwref_res_maps(const cwref_problem* p, double* lat, char* lat_valid, double* apd,
                    char* apd_valid) {
  const auto& L = p->result.lat_map;
  const auto& A = p->result.apd90_map;
  std::memcpy(lat, L.value.data(), L.value.size() * sizeof(double));
  std::memcpy(lat_valid, L.valid.data(), L.valid.size());
  std::memcpy(apd, A.value.data(), A.value.size() * sizeof(double));
  std::memcpy(apd_valid, A.valid.data(), A.valid.size());
}

// ---------------------------------------------------------------- models
int cwref_model_info(const char* name, int* state_count, double* stable_step, double* rest,
                     int rest_cap) {
  try {
    auto m = make_model(name);
    *state_count = m->state_count();
    *stable_step = m->stable_step();
    const auto& r = m->rest_state();
    for (int i = 0; i < rest_cap && i < static_cast<int>(r.size()); ++i)
      rest[i] = r[static_cast<std::size_t>(i)];
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

// Batch rates(): v[n], s[n*ns] (node-major), i_stim[n] -> dv[n], ds[n*ns]
int cwref_rates(const char* name, std::int64_t n, const double* v, const double* s,
                const double* i_stim, double* dv, double* ds) {
  try {
    auto m = make_model(name);
    const int ns = m->state_count();
    for (std::int64_t i = 0; i < n; ++i) {
      double d = 0.0;
      m->rates(v[i], s + i * ns, i_stim[i], d, ds + i * ns);
      dv[i] = d;
    }
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

// pace_to_steady_state: 0 ok, 2 validation, 3 instability (t in fail_t)
int cwref_pace(const char* name, double cycle_ms, int n_beats, double amp, double dur, double* state_out,
               double* apd_out, double* max_rel, double* fail_t, char* msg, int msg_cap) {
  try {
    auto m = make_model(name);
    const PacingResult r = pace_to_steady_state(*m, cycle_ms, n_beats, amp, dur);
    for (std::size_t k = 0; k < r.state.size(); ++k) state_out[k] = r.state[k];
    for (std::size_t b = 0; b < r.apd90_ms.size(); ++b) apd_out[b] = r.apd90_ms[b];
    *max_rel = r.max_rel_change;
    return kOk;
  } catch (const InstabilityError& e) {
    *fail_t = e.time_ms;
    std::snprintf(msg, static_cast<std::size_t>(msg_cap), "%s", e.what());
    return kInstability;
  } catch (const std::exception& e) {
    std::snprintf(msg, static_cast<std::size_t>(msg_cap), "%s", e.what());
    return kValidation;
  }
}

// ---------------------------------------------------------------- postprocess metrics (postprocess.cpp:98-236)
namespace {
Trace make_trace(const double* t, const double* v, std::int64_t n) {
  Trace tr;
  tr.t_ms.assign(t, t + n);
  tr.v_mv.assign(v, v + n);
  return tr;
}
ScalarMap make_map(std::int64_t n, const double* value, const char* valid) {
  ScalarMap m;
  m.value.assign(value, value + n);
  m.valid.assign(valid, valid + n);
  return m;
}
}  // namespace

// 1: APD90 written, 0: none
int cwref_compute_apd90(const double* t, const double* v, std::int64_t n, double* out) {
  const auto r = compute_apd90(make_trace(t, v, n));
  if (r) *out = *r;
  return r ? 1 : 0;
}

int cwref_compute_cv(cwref_problem* p, const double* lat, const char* valid, std::int64_t a, std::int64_t b,
                     double* out) {
  try {
    *out = compute_cv(p->mesh, make_map(p->mesh.node_count(), lat, valid), a, b);
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

int cwref_nrmse(std::int64_t n, const double* rv, const char* rvalid, const double* cv, const char* cvalid,
                double* out) {
  try {
    *out = nrmse(make_map(n, rv, rvalid), make_map(n, cv, cvalid));
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

int cwref_align_and_diff(const double* ta, const double* va, std::int64_t na, const double* tb, const double* vb,
                         std::int64_t nb, double* out) {
  try {
    *out = align_and_diff(make_trace(ta, va, na), make_trace(tb, vb, nb));
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

// ---------------------------------------------------------------- writers (output.cpp, ionic.cpp:13-57)
int cwref_write_vtk_snapshot(cwref_problem* p, const double* v, double t, const char* path) {
  try {
    write_vtk_snapshot(p->mesh, std::vector<double>(v, v + p->mesh.node_count()), t, path);
    return kOk;
  } catch (const std::exception&) {
    return kIo;
  }
}

int cwref_write_map(cwref_problem* p, const double* value, const char* valid, const char* name, int vtk,
                    const char* path) {
  try {
    const ScalarMap m = make_map(p->mesh.node_count(), value, valid);
    if (vtk)
      write_map_vtk(p->mesh, m, name, path);
    else
      write_map_csv(p->mesh, m, path);
    return kOk;
  } catch (const std::exception&) {
    return kIo;
  }
}

int cwref_write_trace_csv(const double* t, const double* v, std::int64_t n, const char* path) {
  try {
    write_trace_csv(make_trace(t, v, n), path);
    return kOk;
  } catch (const std::exception&) {
    return kIo;
  }
}

int cwref_state_save(std::int64_t n, int stride, const double* v, const double* s, const double* last,
                     const std::uint8_t* mon, const char* path) {
  try {
    NodeStateArray a;
    a.n_nodes = n;
    a.stride = stride;
    a.v.assign(v, v + n);
    a.s.assign(s, s + n * stride);
    a.last_dvdt.assign(last, last + n);
    a.model_of_node.assign(mon, mon + n);
    a.save(path);
    return kOk;
  } catch (const std::exception&) {
    return kIo;
  }
}

double cwref_estimate_dt0(const char* name) { return estimate_dt0(*make_model(name)); }

// ---------------------------------------------------------------- rules
int cwref_reaction_substeps(double dvdt, int scheme, int k0_up, int k0_down, int k_max) {
  SchemeConfig c;
  c.scheme = static_cast<Scheme>(scheme);
  c.k0_up = k0_up;
  c.k0_down = k0_down;
  return reaction_substeps(dvdt, c, k_max);
}

int cwref_diffusion_substeps(double dt, double dt_s, int strict, int scheme, int* l, double* dt_ad) {
  try {
    const auto pl = diffusion_substeps(dt, dt_s, strict != 0, static_cast<Scheme>(scheme));
    *l = pl.l;
    *dt_ad = pl.dt_ad;
    return kOk;
  } catch (const std::exception&) {
    return kValidation;
  }
}

int cwref_k_max_for(double dt, const char* name) { return k_max_for(dt, *make_model(name)); }

double cwref_gershgorin(const cwref_problem* p) { return gershgorin_step(p->op); }

// diastolic_threshold with the library defaults except window/dt/duration
double cwref_threshold(const cwref_problem* p, const char* model, const std::int64_t* nodes,
                       std::int64_t n, double window_ms, double duration_ms, double initial_guess,
                       char* err, int errlen) {
  try {
    ThresholdOptions o;
    o.window_ms = window_ms;
    o.duration_ms = duration_ms;
    o.initial_guess = initial_guess;
    std::vector<std::int64_t> sn(nodes, nodes + n);
    return diastolic_threshold(p->mesh, p->op, *make_model(model), sn, o);
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return std::nan("");
  }
}

}  // extern "C"
