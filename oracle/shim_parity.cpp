// TEST INFRASTRUCTURE: the C++ drop-in (include/cardwave_gpu.hpp) side by side
// with the unmodified reference, on the same reference-built problem.
//   shim_parity ap|ord|abort|diffusion   -> one JSON line; exit 0 on parity
//   shim_parity advance|resident          -> StrangIntegrator::advance step by step (resident: device-resident state)
//   shim_parity c2 [t_end_ms]            -> the bench workload (BASELINE configs[1]) end to end
//   shim_parity c1 [t_end_ms]            -> BASELINE configs[0] (ORd-epi, C1 line at 592 mV/ms), default 400 ms
// Built by oracle/Makefile (target `shim`) into oracle/_ref/shim_parity,
// linked against the reference objects and ../paper_2011_04747_b200/libcwgpu.so.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "cardwave/errors.hpp"
#include "cardwave/fem.hpp"
#include "cardwave/mesh.hpp"
#include "cardwave/splitting.hpp"
#include "cardwave/stimulus.hpp"
#include "cardwave_gpu.hpp"

using namespace cardwave;

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "ap";
  const bool c2 = mode == "c2";
  // C2: 5 x 5 cm, h = 0.025, fibres 45 deg, D_l 0.0012 / rho 0.25, ORd-epi, corner disc r = 0.15 at 100 mV/ms
  Mesh mesh = c2 ? build_regular_sheet(5.0, 5.0, 0.025, M_PI / 4) : build_regular_sheet(1.0, 1.0, 0.01, 0.0);
  AssembledOperator op = c2 ? assemble(mesh, build_diffusion_field(mesh, 0.0012, 0.00066, 0.25))
                            : assemble(mesh, build_diffusion_field(mesh, 0.001, 0.00066, 1.0));
  if (mode == "diffusion") {
    std::vector<double> v(op.rows()), a, b;
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = -80.0 + 100.0 * std::sin(0.37 * static_cast<double>(i));
    diffusion_substep(op, v, 0.0123, a);
    gpu::diffusion_substep(op, v, 0.0123, b);
    const bool same = a == b;
    std::printf("{\"mode\":\"diffusion\",\"bitwise\":%s}\n", same ? "true" : "false");
    return same ? 0 : 1;
  }
  const bool ap = mode == "ap";
  std::vector<std::shared_ptr<const CellModel>> models = {make_model(ap ? "aliev-panfilov" : "ohara2011-epi")};
  RegionSelector sel;
  sel.kind = RegionSelector::Kind::half_plane_x_le;
  sel.value = ap ? 0.05 : 0.0;
  if (c2) {
    sel.kind = RegionSelector::Kind::disc;
    sel.cx = 0.0;
    sel.cy = 0.0;
    sel.radius = 0.15;
  }
  Protocol prot;
  Stimulus st;
  st.nodes = select_nodes(mesh, sel);
  st.amplitude = ap || c2 ? 100.0 : 592.0;
  prot.entries.push_back(st);
  ProtocolIndex index(prot, mesh.node_count());
  SimulationSetup setup;
  setup.op = &op;
  setup.models = models;
  setup.protocol = &index;
  setup.probes = {Probe{5050, "mid"}, Probe{10200, "far"}};
  if (c2)
    setup.probes = {Probe{mesh.nearest_node(0.0, 0.0), "corner"}, Probe{mesh.nearest_node(2.5, 2.5), "centre"},
                    Probe{mesh.nearest_node(5.0, 5.0), "far"}};
  SchemeConfig cfg;
  cfg.scheme = Scheme::DAETI;
  cfg.dt_ms = 0.1;
  cfg.t_end_ms = ap ? 100.0 : 20.0;
  if (c2) cfg.t_end_ms = argc > 2 ? std::atof(argv[2]) : 500.0;
  if (mode == "c1") cfg.t_end_ms = argc > 2 ? std::atof(argv[2]) : 400.0;
  cfg.k0_down = mode == "abort" ? 1 : (ap ? 1 : 3);
  NodeStateArray s0 = make_initial_state(mesh, models, {0});
  if (mode == "advance" || mode == "resident") {
    // StrangIntegrator::advance step by step (oracles::reference_solution-style callers): the reference
    // and the drop-in side by side, V compared after every step (ORd, C1 line, k0_down = 3, 20 ms);
    // "resident": the drop-in keeps the state on the device (set_state_residency), the cell states come
    // back at the end through sync_state()
    cfg.t_end_ms = 20.0;
    StrangIntegrator ref(setup, cfg);
    gpu::StrangIntegrator dev(setup, cfg);
    if (mode == "resident") dev.set_state_residency(true);
    NodeStateArray sa = s0, sb = s0;
    const std::int64_t n_steps = static_cast<std::int64_t>(std::ceil(cfg.t_end_ms / cfg.dt_ms - 1e-9));
    double dv = 0.0;
    for (std::int64_t k = 0; k < n_steps; ++k) {
      ref.advance(sa, k * cfg.dt_ms, k, n_steps);
      dev.advance(sb, k * cfg.dt_ms, k, n_steps);
      for (std::size_t i = 0; i < sa.v.size(); ++i) dv = std::max(dv, std::abs(sa.v[i] - sb.v[i]));
    }
    if (mode == "resident") dev.sync_state(sb);
    double ds = 0.0;
    for (std::size_t i = 0; i < sa.s.size(); ++i) ds = std::max(ds, std::abs(sa.s[i] - sb.s[i]) / (1.0 + std::abs(sa.s[i])));
    const bool kh = ref.k_histogram() == dev.k_histogram();
    const bool pass = dv <= 1e-6 && ds <= 1e-9 && kh;
    std::printf("{\"mode\":\"%s\",\"steps\":%lld,\"max_dV_mV\":%.3e,\"max_rel_dstate\":%.3e,\"khist_equal\":%s,"
                "\"pass\":%s}\n",
                mode.c_str(), static_cast<long long>(n_steps), dv, ds, kh ? "true" : "false", pass ? "true" : "false");
    return pass ? 0 : 1;
  }
  // snapshots (asynchronous in the drop-in) and progress callbacks
  std::vector<std::pair<double, std::vector<double>>> snaps[2];
  int which = 0;
  long progress_calls[2] = {0, 0};
  setup.snapshot_interval_ms = ap ? 5.0 : (mode == "abort" ? 0.5 : 2.0);
  setup.on_snapshot = [&](double t, const std::vector<double>& v) { snaps[which].emplace_back(t, v); };
  setup.progress_every = 37;
  setup.on_progress = [&](std::int64_t, double, const TimingBreakdown&) { ++progress_calls[which]; };

  long ref_node = -1, gpu_node = -1;
  double ref_t = 0, gpu_t = 0;
  SimulationResult a, b;
  bool ref_ok = true, gpu_ok = true;
  try {
    a = run_simulation(s0, setup, cfg);
  } catch (const InstabilityError& e) {
    ref_ok = false;
    ref_node = e.node_index;
    ref_t = e.time_ms;
  }
  which = 1;
  try {
    b = gpu::run_simulation(s0, setup, cfg);
  } catch (const InstabilityError& e) {
    gpu_ok = false;
    gpu_node = e.node_index;
    gpu_t = e.time_ms;
  }
  // snapshot series: same count and times; V bit-exact for AP, <= 1e-6 mV for ORd
  bool snaps_same = snaps[0].size() == snaps[1].size() && progress_calls[0] == progress_calls[1];
  double snap_dv = 0.0;
  for (std::size_t k = 0; snaps_same && k < snaps[0].size(); ++k) {
    snaps_same = snaps[0][k].first == snaps[1][k].first;
    for (std::size_t i = 0; i < snaps[0][k].second.size(); ++i)
      snap_dv = std::max(snap_dv, std::abs(snaps[0][k].second[i] - snaps[1][k].second[i]));
  }
  // (abort mode: the last snapshots precede a blow-up, where ulp differences
  // are amplified without bound -- there only count and times are compared)
  if (mode != "abort") snaps_same = snaps_same && (ap ? snap_dv == 0.0 : snap_dv <= 1e-6);
  if (!ref_ok || !gpu_ok) {
    const bool same = !ref_ok && !gpu_ok && ref_node == gpu_node && ref_t == gpu_t && snaps_same;
    std::printf("{\"mode\":\"%s\",\"ref_abort\":[%ld,%.17g],\"gpu_abort\":[%ld,%.17g],\"snapshots\":[%zu,%zu],"
                "\"match\":%s}\n",
                mode.c_str(), ref_node, ref_t, gpu_node, gpu_t, snaps[0].size(), snaps[1].size(),
                same ? "true" : "false");
    return same ? 0 : 1;
  }
  double dv = 0, dl = 0;
  for (std::size_t i = 0; i < a.final_state.v.size(); ++i) dv = std::max(dv, std::abs(a.final_state.v[i] - b.final_state.v[i]));
  for (std::size_t p = 0; p < a.traces.size(); ++p)
    for (std::size_t q = 0; q < a.traces[p].v_mv.size(); ++q)
      dv = std::max(dv, std::abs(a.traces[p].v_mv[q] - b.traces[p].v_mv[q]));
  bool valid_same = a.lat_map.valid == b.lat_map.valid;
  for (std::size_t i = 0; i < a.lat_map.value.size(); ++i)
    if (a.lat_map.valid[i]) dl = std::max(dl, std::abs(a.lat_map.value[i] - b.lat_map.value[i]));
  const bool kh = a.k_histogram == b.k_histogram;
  const bool pass = snaps_same && (ap ? (dv == 0.0 && dl == 0.0 && kh && valid_same)
                                       : (dv <= 1e-6 && dl < 1e-6 && kh && valid_same));
  std::printf("{\"mode\":\"%s\",\"max_dV_mV\":%.3e,\"max_dLAT_ms\":%.3e,\"khist_equal\":%s,\"lat_valid_equal\":%s,"
              "\"snapshots\":[%zu,%zu],\"snapshot_max_dV\":%.3e,\"progress_calls\":[%ld,%ld],"
              "\"pass\":%s,\"ref_ms\":%.1f,\"gpu_ms\":%.1f}\n",
              mode.c_str(), dv, dl, kh ? "true" : "false", valid_same ? "true" : "false", snaps[0].size(),
              snaps[1].size(), snap_dv, progress_calls[0], progress_calls[1], pass ? "true" : "false",
              a.timing.total_ms, b.timing.total_ms);
  return pass ? 0 : 1;
}
