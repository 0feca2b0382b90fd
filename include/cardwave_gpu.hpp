// cardwave_gpu.hpp -- header-only C++ drop-in for the reference's hot path.
//
// Include after the reference headers (cardwave/splitting.hpp) and link
// libcwgpu.so. The three entry points carry the reference's own signatures
// and semantics:
//
//   cardwave::gpu::StrangIntegrator   <-  cardwave::StrangIntegrator  (splitting.hpp:101-127)
//   cardwave::gpu::run_simulation     <-  cardwave::run_simulation    (splitting.hpp:139-140)
//   cardwave::gpu::diffusion_substep  <-  cardwave::diffusion_substep (fem.hpp:56-57)
//
// Errors are rethrown as the reference's exception types (errors.hpp):
// ValidationError, InstabilityError(node, t_ms), IoError; CUDA failures as
// std::runtime_error. There is no CPU fallback: a model the device path does
// not implement (CellModel::name() outside the registry) is a ValidationError.
//
// Multi-GPU (one process per GPU, y-slabs, NCCL halo exchange): pass a
// gpu::Placement{device, rank, world, nccl_id}; every rank constructs the
// integrator with the full problem and run_simulation returns the global
// SimulationResult on every rank (cwg_gather_result).
//
// State residency (StrangIntegrator::advance): by default every advance()
// uploads and downloads the whole NodeStateArray, exactly the reference's
// in-place semantics (splitting.cpp:171-181) for any caller. A caller that
// steps one state object through many advance() calls and reads only V
// between them can call set_state_residency(true): the state then stays on
// the device, is uploaded only when advance() sees other buffers (or after
// mark_state_modified()), V and last_dvdt come back every step (8 + 8 B per
// node instead of 344 for ORd), and the cell states on sync_state() or on
// an InstabilityError.
//
// ProtocolIndex exposes no accessors (stimulus.hpp:35-50), so the shim reads
// its two members through a layout mirror, guarded by static_asserts; a
// maintainer who prefers can instead add `entries()`/`node_entries()`
// accessors to the reference and replace detail::protocol_view.
#ifndef CARDWAVE_GPU_HPP
#define CARDWAVE_GPU_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cardwave/errors.hpp"
#include "cardwave/fem.hpp"
#include "cardwave/ionic.hpp"
#include "cardwave/splitting.hpp"
#include "cardwave/stimulus.hpp"
#include "cwgpu.h"

namespace cardwave::gpu {

/// Device placement of an integrator: one GPU (default), or rank `rank` of a
/// `world`-rank y-slab run whose ranks share one NCCL unique id (128 bytes).
struct Placement {
  int device = 0;
  int rank = 0;
  int world = 1;
  const unsigned char* nccl_id = nullptr;
};

namespace detail {

[[noreturn]] inline void rethrow(int rc, const cwg_error& e) {
  std::string msg(e.msg);
  if (rc == CWG_EVALIDATION) throw ValidationError(msg);
  if (rc == CWG_EINSTABILITY) {
    // cwg_error.msg already carries " (node N, t = T ms)"; InstabilityError appends its own
    const auto cut = msg.find(" (node ");
    throw InstabilityError(cut == std::string::npos ? msg : msg.substr(0, cut), static_cast<long>(e.node),
                           e.t_ms);
  }
  if (rc == CWG_EIO) throw IoError(msg);
  throw std::runtime_error("cwgpu: " + msg);
}

inline void check(int rc, const cwg_error& e) {
  if (rc != CWG_OK) rethrow(rc, e);
}

inline void check(int rc) {
  if (rc != CWG_OK) {
    cwg_error e{};
    e.code = rc;
    std::snprintf(e.msg, sizeof(e.msg), "%s", "cwgpu call failed");
    rethrow(rc, e);
  }
}

// Layout mirror of ProtocolIndex's private members (stimulus.hpp:43-48).
struct ProtocolMirror {
  struct Entry {
    double t_start, duration, amplitude;
    std::optional<double> period;
  };
  std::vector<Entry> entries_;
  std::vector<std::vector<std::int32_t>> node_entries_;
};
static_assert(sizeof(ProtocolMirror) == sizeof(ProtocolIndex), "ProtocolIndex layout changed");

struct FlatProtocol {
  std::vector<double> t0, dur, amp, per;
  std::vector<std::int32_t> ptr, ids;
};

inline FlatProtocol protocol_view(const ProtocolIndex* pi, std::int64_t n) {
  FlatProtocol f;
  f.ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  if (!pi) return f;
  const auto* m = reinterpret_cast<const ProtocolMirror*>(pi);
  for (const auto& e : m->entries_) {
    f.t0.push_back(e.t_start);
    f.dur.push_back(e.duration);
    f.amp.push_back(e.amplitude);
    f.per.push_back(e.period ? *e.period : std::nan(""));
  }
  for (std::int64_t i = 0; i < n; ++i) {
    for (auto id : m->node_entries_[static_cast<std::size_t>(i)]) f.ids.push_back(id);
    f.ptr[static_cast<std::size_t>(i) + 1] = static_cast<std::int32_t>(f.ids.size());
  }
  return f;
}

inline int model_kind(const CellModel& m) {
  const int k = cwg_model_kind_from_name(m.name().c_str());
  if (k < 0) throw ValidationError("gpu: no device implementation of cell model '" + m.name() + "'");
  return k;
}

// Owns the device context; created lazily because model_of_node arrives with
// the state (the reference ctor sees only setup + cfg).
class Context {
 public:
  Context(const SimulationSetup& setup, const SchemeConfig& cfg, const Placement& pl)
      : setup_(setup), cfg_(cfg), device_(pl.device), place_(pl) {
    cfg.validate();
    if (setup.op == nullptr) throw ValidationError("integrator: missing assembled operator");
    if (setup.models.empty()) throw ValidationError("integrator: no cell models");
    for (const auto& m : setup.models) kinds_.push_back(model_kind(*m));
    dt_eff_ = cfg.scheme == Scheme::OSTAR ? std::min(cfg.dt_ms, setup.op->dt_s) : cfg.dt_ms;
    plan_ = diffusion_substeps(dt_eff_, setup.op->dt_s, cfg.strict_substeps, cfg.scheme);
    for (const auto& m : setup.models) k_max_global_ = std::max(k_max_global_, k_max_for(dt_eff_, *m));
    khist_.assign(static_cast<std::size_t>(k_max_global_) + 1, 0);
  }
  ~Context() {
    if (ctx_) cwg_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  cwg_ctx* get(const NodeStateArray& state) {
    if (ctx_) return ctx_;
    const AssembledOperator& op = *setup_.op;
    const std::int64_t n = op.rows();
    if (state.n_nodes != n) throw ValidationError("integrator: state does not match the operator");
    flat_ = protocol_view(setup_.protocol, n);
    probes_.clear();
    for (const auto& p : setup_.probes) probes_.push_back(p.node);
    cwg_problem p{};
    p.n = n;
    p.row_ptr = op.row_ptr.data();
    p.col = op.col.data();
    p.val = op.val.data();
    p.lumped_mass = op.lumped_mass.data();
    p.dt_s = op.dt_s;
    p.op_kind = CWG_OP_AUTO;
    p.n_models = static_cast<int>(kinds_.size());
    p.model_kind = kinds_.data();
    p.model_of_node = state.model_of_node.data();
    p.n_stim = static_cast<int>(flat_.t0.size());
    if (p.n_stim) {
      p.stim_t_start = flat_.t0.data();
      p.stim_duration = flat_.dur.data();
      p.stim_amplitude = flat_.amp.data();
      p.stim_period = flat_.per.data();
      p.stim_node_ptr = flat_.ptr.data();
      p.stim_ids = flat_.ids.data();
    }
    p.n_probes = static_cast<int>(probes_.size());
    p.probes = probes_.data();
    p.lat_threshold_mv = setup_.lat_threshold_mv;
    p.map_interval_ms = setup_.map_interval_ms;
    p.scheme = static_cast<int>(cfg_.scheme);
    p.dt_ms = cfg_.dt_ms;
    p.t_end_ms = cfg_.t_end_ms;
    p.k0_up = cfg_.k0_up;
    p.k0_down = cfg_.k0_down;
    p.strict_substeps = cfg_.strict_substeps ? 1 : 0;
    p.record_interval_ms = cfg_.record_interval_ms;
    p.device = device_;
    p.rank = place_.rank;
    p.world = place_.world;
    p.nccl_id = place_.nccl_id;
    cwg_error e{};
    check(cwg_create(&p, &ctx_, &e), e);
    return ctx_;
  }

  const SimulationSetup& setup_;
  const SchemeConfig& cfg_;
  int device_;
  Placement place_;
  std::vector<int> kinds_;
  double dt_eff_ = 0.0;
  DiffusionPlan plan_;
  int k_max_global_ = 1;
  std::vector<std::int64_t> khist_;
  TimingBreakdown timing_;
  FlatProtocol flat_;
  std::vector<std::int64_t> probes_;
  cwg_ctx* ctx_ = nullptr;
};

}  // namespace detail

/// Drop-in for cardwave::StrangIntegrator (splitting.hpp:101-127).
class StrangIntegrator {
 public:
  StrangIntegrator(const SimulationSetup& setup, const SchemeConfig& cfg, int device = 0)
      : StrangIntegrator(setup, cfg, Placement{device, 0, 1, nullptr}) {}
  StrangIntegrator(const SimulationSetup& setup, const SchemeConfig& cfg, const Placement& pl)
      : c_(std::make_unique<detail::Context>(setup, cfg, pl)) {}

  /// One outer step; mutates `state` in place like splitting.cpp:171-181.
  void advance(NodeStateArray& state, double t_ms, std::int64_t step_index, std::int64_t n_steps) {
    cwg_ctx* ctx = c_->get(state);
    const bool same = resident_ && !dirty_ && state.v.data() == synced_v_ && state.s.data() == synced_s_ &&
                      state.last_dvdt.data() == synced_last_;
    if (!same)
      detail::check(cwg_upload_state(ctx, state.v.data(), state.s.data(), state.stride, state.last_dvdt.data()));
    cwg_error e{};
    const int rc = cwg_advance(ctx, t_ms, step_index, n_steps, &e);
    const bool full = !resident_ || rc != CWG_OK;
    detail::check(cwg_download_state(ctx, state.v.data(), full ? state.s.data() : nullptr, state.stride,
                                     state.last_dvdt.data()));
    synced_v_ = state.v.data();
    synced_s_ = state.s.data();
    synced_last_ = state.last_dvdt.data();
    dirty_ = false;
    refresh();
    detail::check(rc, e);
  }

  /// Opt-in device residency of the state across advance() calls (see the header comment).
  void set_state_residency(bool on) {
    resident_ = on;
    dirty_ = true;
  }
  /// The caller changed the state's values in place: the next advance() uploads it.
  void mark_state_modified() { dirty_ = true; }
  /// Bring the cell states (and V, last_dvdt) of a resident run back to `state`.
  void sync_state(NodeStateArray& state) {
    if (!c_->ctx_) return;
    detail::check(cwg_download_state(c_->ctx_, state.v.data(), state.s.data(), state.stride,
                                     state.last_dvdt.data()));
  }

  double dt_effective() const { return c_->dt_eff_; }
  const DiffusionPlan& plan() const { return c_->plan_; }
  int k_max_global() const { return c_->k_max_global_; }
  const std::vector<std::int64_t>& k_histogram() const { return c_->khist_; }
  const TimingBreakdown& timing() const { return c_->timing_; }

  cwg_ctx* handle(const NodeStateArray& state) { return c_->get(state); }
  void refresh() {
    if (!c_->ctx_) return;
    cwg_get_khist(c_->ctx_, c_->khist_.data(), static_cast<int>(c_->khist_.size()));
    cwg_get_timing(c_->ctx_, &c_->timing_.reaction_ms, &c_->timing_.diffusion_ms, &c_->timing_.recording_ms);
  }
  int world() const { return c_->place_.world; }

 private:
  std::unique_ptr<detail::Context> c_;
  bool resident_ = false, dirty_ = true;
  const double *synced_v_ = nullptr, *synced_s_ = nullptr, *synced_last_ = nullptr;
};

/// Drop-in for cardwave::run_simulation (splitting.cpp:219-294): device-resident
/// state, CUDA-graph replay between record points, callbacks at their cadence.
inline SimulationResult run_simulation(NodeStateArray state, const SimulationSetup& setup,
                                       const SchemeConfig& cfg, const Placement& place = Placement{}) {
  const auto t_run0 = std::chrono::steady_clock::now();
  StrangIntegrator integ(setup, cfg, place);
  cwg_ctx* ctx = integ.handle(state);
  cwg_info info{};
  cwg_get_info(ctx, &info);
  detail::check(cwg_upload_state(ctx, state.v.data(), state.s.data(), state.stride, state.last_dvdt.data()));
  detail::check(cwg_run_begin(ctx));
  const std::int64_t n_steps = info.n_steps;
  const double dt = info.dt_effective;
  const std::int64_t every_snap =
      setup.snapshot_interval_ms > 0.0 && setup.on_snapshot
          ? std::max<std::int64_t>(1, std::llround(setup.snapshot_interval_ms / dt))
          : 0;
  const std::int64_t every_prog = setup.progress_every > 0 && setup.on_progress ? setup.progress_every : 0;
  if (every_snap) setup.on_snapshot(0.0, state.v);
  // Snapshots are asynchronous: the V copy of snapshot N is enqueued after the
  // steps up to it, the next chunk of steps is enqueued, and only then does
  // the host wait for the copy and run on_snapshot -- the callback (e.g. the
  // reference's write_vtk_snapshot) overlaps the device computing the next
  // chunk. cwg_snapshot_wait reports a failure that happened before the
  // snapshot point, so no snapshot after the reference's throw is delivered.
  std::vector<double> snap;
  bool registered = false;
  if (every_snap) {
    snap.assign(state.v.size(), 0.0);
    registered = cwg_host_register(snap.data(), snap.size() * sizeof(double)) == CWG_OK;
  }
  struct Unregister {
    bool on;
    double* p;
    ~Unregister() {
      if (on) cwg_host_unregister(p);
    }
  } unreg{registered, snap.data()};
  bool pending = false;
  double pending_t = 0.0;
  std::int64_t s = 0;
  cwg_error e{};
  auto deliver = [&] {
    const int rc = cwg_snapshot_wait(ctx, &e);
    if (rc != CWG_OK) detail::rethrow(rc, e);
    pending = false;
    setup.on_snapshot(pending_t, snap);
  };
  while (s < n_steps) {
    std::int64_t next = n_steps;
    if (every_snap) next = std::min(next, (s / every_snap + 1) * every_snap);
    if (every_prog) next = std::min(next, (s / every_prog + 1) * every_prog);
    detail::check(cwg_run_steps(ctx, s, next - s));
    if (pending) deliver();
    s = next;
    if (every_snap && s % every_snap == 0) {
      detail::check(cwg_snapshot_begin(ctx, snap.data()));
      pending = true;
      pending_t = static_cast<double>(s) * dt;
    }
    if ((every_prog && s % every_prog == 0) || s == n_steps) {
      if (pending) deliver();
      const int rc = cwg_run_sync(ctx, &e);
      if (rc != CWG_OK) detail::rethrow(rc, e);
      if (every_prog && s % every_prog == 0) {
        integ.refresh();
        TimingBreakdown tb = integ.timing();
        tb.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_run0).count();
        setup.on_progress(s, static_cast<double>(s) * dt, tb);
      }
    }
  }
  if (pending) deliver();
  SimulationResult r;
  r.dt_effective = dt;
  r.dt_s = setup.op->dt_s;
  r.plan = integ.plan();
  r.n_steps = n_steps;
  const std::size_t ns = static_cast<std::size_t>(info.n_samples);
  std::vector<double> t(ns), v(ns * std::max<std::size_t>(setup.probes.size(), 1));
  detail::check(cwg_get_traces(ctx, t.data(), v.data()));
  for (std::size_t p = 0; p < setup.probes.size(); ++p) {
    Trace tr;
    tr.node = setup.probes[p].node;
    tr.name = setup.probes[p].name;
    tr.t_ms = t;
    tr.v_mv.assign(v.begin() + static_cast<std::ptrdiff_t>(p * ns), v.begin() + static_cast<std::ptrdiff_t>((p + 1) * ns));
    r.traces.push_back(std::move(tr));
  }
  const std::size_t n = static_cast<std::size_t>(state.n_nodes);
  r.lat_map.value.resize(n);
  r.apd90_map.value.resize(n);
  std::vector<std::uint8_t> lv(n), av(n);
  // the global maps and final state on every rank (world == 1: the plain download)
  detail::check(cwg_gather_result(ctx, state.v.data(), state.s.data(), state.stride, state.last_dvdt.data(),
                                  r.lat_map.value.data(), lv.data(), r.apd90_map.value.data(), av.data()));
  r.lat_map.valid.assign(lv.begin(), lv.end());
  r.apd90_map.valid.assign(av.begin(), av.end());
  integ.refresh();
  r.k_histogram = integ.k_histogram();
  r.timing = integ.timing();
  r.timing.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_run0).count();
  r.final_state = std::move(state);
  return r;
}

/// Drop-in for cardwave::diffusion_substep (fem.cpp:194-207), bit-identical.
inline void diffusion_substep(const AssembledOperator& op, const std::vector<double>& v, double dt_sub,
                              std::vector<double>& out, int device = 0) {
  out.resize(v.size());
  cwg_error e{};
  detail::check(cwg_diffusion_substep(op.rows(), op.row_ptr.data(), op.col.data(), op.val.data(),
                                      op.lumped_mass.data(), v.data(), dt_sub, out.data(), device, &e),
                e);
}

}  // namespace cardwave::gpu

#endif
