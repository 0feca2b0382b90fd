"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bit-exact where the reference arithmetic allows it (integer rules,
diffusion, Aliev-Panfilov, the detector); ORd/MacCannell go through libdevice
exp/log instead of glibc's, so they are held to the fp64 tolerance of
north_star: max|dV| <= 1e-6 mV on traces and the final field, identical
k-histogram, identical LAT rank order on the sampled node set.
"""
import math

import numpy as np
import pytest

from helpers import gpu_run, lat_order_equal, oracle_run, run_both

pytestmark = pytest.mark.gpu

V_TOL_MV = 1e-6  # north_star: max|dV| <= 1e-6 mV


@pytest.fixture(scope="module")
def cw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    return cw


@pytest.fixture(scope="module")
def problems(cw):
    from paper_2011_04747_b200 import problems
    return problems


def _states(rest, n, rng, spread):
    ns = len(rest) - 1
    s = np.tile(rest[1:], (n, 1)) * rng.uniform(1 - spread, 1 + spread, (n, ns))
    return s


@pytest.mark.parametrize("model", ["aliev-panfilov", "maccannell2007", "ohara2011-endo", "ohara2011-epi",
                                   "ohara2011-mid"])
def test_rates_against_oracle(cw, ora, model):
    rng = np.random.default_rng(1)
    m = cw.make_model(model)
    rest = m.rest_state()
    assert np.array_equal(rest, ora.rest_state(model))
    n = 4096
    v = rng.uniform(-95.0, 45.0, n) if model != "aliev-panfilov" else rng.uniform(-85.0, 25.0, n)
    s = _states(rest, n, rng, 0.3) if model != "aliev-panfilov" else rng.uniform(0.0, 2.0, (n, 1))
    ist = rng.choice([0.0, 80.0], n)
    dv_g, ds_g = m.rates(v, s, ist)
    dv_o, ds_o = ora.rates(model, v, s, ist)
    if model == "aliev-panfilov":
        assert np.array_equal(dv_g, dv_o) and np.array_equal(ds_g, ds_o)
    else:
        scale_v = np.maximum(1.0, np.abs(dv_o))
        assert np.max(np.abs(dv_g - dv_o) / scale_v) < 1e-11
        scale_s = np.maximum(np.abs(ds_o), 1e-300) + 1e-9 * np.max(np.abs(ds_o), axis=0)
        assert np.max(np.abs(ds_g - ds_o) / scale_s) < 1e-9


@pytest.mark.parametrize("which", ["c1", "c2", "fib"])
def test_diffusion_substep_bitwise(cw, ora, which):
    rng = np.random.default_rng(2)
    if which == "c1":
        sh = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0)
    elif which == "c2":
        sh = cw.Sheet(5.0, 5.0, 0.025, math.pi / 4, d0_myocyte=0.0012, rho=0.25)
    else:
        sh = cw.Sheet(2.0, 1.0, 0.02, 0.7, fib_fraction=0.3, seed=11)
    op = sh.op
    v = rng.uniform(-90.0, 40.0, sh.n)
    out_g = cw.diffusion_substep(op, v, 0.01)
    out_o = ora.diffusion_substep((op.row_ptr, op.col, op.val, op.lumped_mass), v, 0.01)
    assert np.array_equal(out_g, out_o)


def _compare_exact(res, o):
    assert np.array_equal(res.final_state.v, o["v"])
    assert np.array_equal(res.final_state.s.reshape(o["s"].shape), o["s"])
    assert np.array_equal(res.final_state.last_dvdt, o["last_dvdt"])
    assert np.array_equal(res.k_histogram, o["k_histogram"])
    for q, tr in enumerate(res.traces):
        assert np.array_equal(tr.v_mv, o["traces"][q])
        assert np.array_equal(tr.t_ms, o["trace_t"])
    assert np.array_equal(res.lat_map.valid, o["lat_valid"])
    assert np.array_equal(res.lat_map.value[o["lat_valid"]], o["lat"][o["lat_valid"]])
    assert np.array_equal(res.apd90_map.valid, o["apd_valid"])
    assert np.array_equal(res.apd90_map.value[o["apd_valid"]], o["apd90"][o["apd_valid"]])


def _compare_tol(res, o, nx1, probes=()):
    import orapy
    import paper_2011_04747_b200 as cw
    if isinstance(o, orapy.OracleInstability):  # the reference aborts: so must we, at the same node and time
        assert isinstance(res, cw.InstabilityError), "oracle aborted, GPU did not"
        assert (res.node_index, res.time_ms) == (o.node, o.t)
        return
    assert not isinstance(res, Exception), f"GPU aborted, oracle did not: {res}"
    dv = np.max(np.abs(res.final_state.v - o["v"]))
    print(f"max|dV| final = {dv:.3e} mV")
    assert dv <= V_TOL_MV, f"final V differs by {dv} mV"
    for q, tr in enumerate(res.traces):
        d = np.max(np.abs(tr.v_mv - o["traces"][q]))
        assert d <= V_TOL_MV, f"trace {q} differs by {d} mV"
    assert np.array_equal(res.k_histogram, o["k_histogram"])
    assert np.array_equal(res.lat_map.valid, o["lat_valid"])
    lv = o["lat_valid"]
    if lv.any():
        dl = np.max(np.abs(res.lat_map.value[lv] - o["lat"][lv]))
        print(f"max|dLAT| = {dl:.3e} ms")
        assert dl < 1e-6
    assert lat_order_equal(res.lat_map.value, res.lat_map.valid, o["lat"], o["lat_valid"], nx1, probes)


def test_c1_aliev_panfilov_bitwise(cw, ora, problems):
    p = problems.c1(model="aliev-panfilov", t_end=120.0, k0_down=1)
    res = gpu_run(p)
    o = oracle_run(p)
    _compare_exact(res, o)
    assert res.lat_map.valid.sum() > 0.9 * p.n  # the wave crossed the sheet


def test_c1_ord_epi_tolerance(cw, ora, problems):
    p = problems.c1(t_end=30.0)
    res, o = run_both(p)
    _compare_tol(res, o, p.sheet.nx1, p.probes)
    assert res.lat_map.valid.sum() > 100


def test_unstable_strip_aborts_like_oracle(cw, ora, problems):
    """Any abort must reproduce the oracle's (node, t); here a strong fibrotic-sheet stimulus."""
    from paper_2011_04747_b200 import api
    sh = cw.Sheet(1.0, 0.5, 0.02, 0.3, d0_myocyte=0.0017, d0_fibrotic=0.00066, rho=0.25, fib_fraction=0.2, seed=5)
    nodes = sh.select("x_le", value=0.05)
    prob = problems.Problem("fib", sh, ["ohara2011-epi", "maccannell2007"], sh.tags.astype(np.uint8),
                            [(nodes, 0.0, 1.0, 150.0, None)], api.SchemeConfig(dt_ms=0.1, t_end_ms=5.0, k0_down=3),
                            [0])
    res, o = run_both(prob)
    _compare_tol(res, o, sh.nx1)


def test_c1_ord_abort_fixture(cw, ora, problems):
    """Paper k0 (k0_down = 1) aborts in the reference at node 16, t = 2.04 ms."""
    p = problems.c1(t_end=10.0, k0_down=1)
    with pytest.raises(ora.OracleInstability) as eo:
        oracle_run(p)
    with pytest.raises(cw.InstabilityError) as eg:
        gpu_run(p)
    assert eg.value.node_index == eo.value.node == 16
    assert eg.value.time_ms == eo.value.t
    assert abs(eg.value.time_ms - 2.04) < 1e-9


@pytest.mark.parametrize("scheme,dt", [("OST", 0.01), ("OSTAR", 0.1)])
def test_schemes_ap_bitwise(cw, ora, problems, scheme, dt):
    p = problems.c1(model="aliev-panfilov", t_end=15.0, scheme=cw.Scheme[scheme], dt=dt)
    res = gpu_run(p)
    o = oracle_run(p)
    _compare_exact(res, o)


def test_daeti_reduces_to_ostar_bitwise(cw, problems):
    """with dt/2 <= dt_s and k_max = 1, DAETI == OSTAR bit for bit."""
    from paper_2011_04747_b200 import api
    sh = cw.Sheet(2.0, 2.0, 0.02, math.pi / 4, d0_myocyte=0.0012, rho=0.25)
    nodes = sh.select("x_le", value=0.05)
    out = []
    for scheme in (api.Scheme.DAETI, api.Scheme.OSTAR):
        prob = problems.Problem("red", sh, ["aliev-panfilov"], np.zeros(sh.n, np.uint8),
                                [(nodes, 0.0, 1.0, 100.0, None)],
                                api.SchemeConfig(scheme=scheme, dt_ms=0.05, t_end_ms=30.0), [0, sh.n // 2])
        assert 0.05 / 2 <= sh.op.dt_s
        out.append(gpu_run(prob))
    a, b = out
    assert np.array_equal(a.final_state.v, b.final_state.v)
    assert np.array_equal(a.traces[1].v_mv, b.traces[1].v_mv)
    assert np.array_equal(a.lat_map.value[a.lat_map.valid], b.lat_map.value[b.lat_map.valid])


def test_advance_matches_graph_run(cw, problems):
    """StrangIntegrator::advance step by step == the graph-replayed run_simulation."""
    p = problems.c1(model="ohara2011-epi", t_end=6.0)
    setup = p.setup()
    st = p.initial_state()
    integ = cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node)
    n_steps = integ.info.n_steps
    for step in range(n_steps):
        integ.advance(st, step * integ.dt_effective(), step, n_steps, sync_state=(step == n_steps - 1))
    res = gpu_run(p)
    assert np.array_equal(st.v, res.final_state.v)
    assert np.array_equal(st.s, res.final_state.s)
    assert np.array_equal(integ.k_histogram(), res.k_histogram)


def test_periodic_stimulus_ap_bitwise(cw, ora, problems):
    p = problems.c1(model="aliev-panfilov", t_end=40.0)
    nodes = p.stimuli[0][0]
    p.stimuli = [(nodes, 2.0, 1.5, 90.0, 17.0), (nodes[:5], 0.0, 1.0, 50.0, None)]
    res = gpu_run(p)
    o = oracle_run(p)
    _compare_exact(res, o)


def test_fibrosis_two_models(cw, ora, problems):
    """Fibroblast-tagged nodes run MacCannell, myocytes ORd-epi (model bins)."""
    from paper_2011_04747_b200 import api
    sh = cw.Sheet(1.0, 0.5, 0.02, 0.3, d0_myocyte=0.0017, d0_fibrotic=0.00066, rho=0.25, fib_fraction=0.2, seed=5)
    nodes = sh.select("x_le", value=0.05)
    prob = problems.Problem("fib", sh, ["ohara2011-epi", "maccannell2007"], sh.tags.astype(np.uint8),
                            [(nodes, 0.0, 1.0, 80.0, None)], api.SchemeConfig(dt_ms=0.1, t_end_ms=12.0, k0_down=3),
                            [0, sh.n - 1])
    res, o = run_both(prob)
    _compare_tol(res, o, sh.nx1)
    assert not isinstance(res, Exception)


def test_c2_short(cw, ora, problems):
    p = problems.c2(t_end=8.0)
    res, o = run_both(p)
    _compare_tol(res, o, p.sheet.nx1, p.probes)
    assert not isinstance(res, Exception)


def test_c3_extension_small(cw, ora, problems):
    """Scar / border zone / passive nodes / GKr jitter (extension; oracle-pinned only)."""
    p = problems.c3(t_end=12.0, h=0.05, size=5.0, amplitude=100.0)
    res, o = run_both(p)
    _compare_tol(res, o, p.sheet.nx1, p.probes)
    assert not isinstance(res, Exception)


def test_launches_counted(cw, problems):
    p = problems.c1(model="aliev-panfilov", t_end=3.0)
    integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=p.model_of_node)
    integ.upload(p.initial_state())
    integ.run_begin()
    integ.run_steps(0, integ.info.n_steps)
    integ.run_sync()
    assert integ.launch_count() > integ.info.n_steps


# ----------------------------------------------------------------------------- 3D slabs (extension)
def test_slab3d_aliev_panfilov_bitwise(cw, ora, problems):
    """Structured 27-point operator + reaction vs the oracle's independent CSR assembly: bit-exact."""
    p = problems.slab(0.4, 0.3, 0.2, 0.02, model="aliev-panfilov", t_end=20.0, amplitude=100.0)
    res = gpu_run(p)
    o = oracle_run(p)
    _compare_exact(res, o)


def test_slab3d_ord_sites_tolerance(cw, ora, problems):
    p = problems.slab(0.6, 0.4, 0.2, 0.02, t_end=8.0, stim="sites", n_sites=3, site_radius=0.1, amplitude=150.0)
    res, o = run_both(p)
    _compare_tol(res, o, p.sheet.nx1, p.probes)


# ----------------------------------------------------------------------------- callbacks (splitting.cpp:265-283)
def test_async_snapshots_bitwise(cw, ora, problems):
    """on_snapshot receives V at every snapshot time, bit-identical to the oracle
    run stopped at that time; on_progress fires at its cadence."""
    p = problems.c1(model="aliev-panfilov", t_end=20.0, k0_down=1)
    setup = p.setup()
    snaps, prog = [], []
    setup.snapshot_interval_ms = 2.0
    setup.on_snapshot = lambda t, v: snaps.append((t, v))
    setup.progress_every = 45
    setup.on_progress = lambda step, t, tb: prog.append(step)
    res = cw.run_simulation(p.initial_state(), setup, p.cfg)
    assert [round(t, 9) for t, _ in snaps] == [round(2.0 * k, 9) for k in range(11)]
    assert prog == [45, 90, 135, 180]
    assert np.array_equal(snaps[-1][1], res.final_state.v)
    o = oracle_run(p, snapshot_interval=2.0)
    assert len(o["snapshots"]) == len(snaps)
    for (tg, vg), (to, vo) in zip(snaps, o["snapshots"]):
        assert tg == to and np.array_equal(vg, vo), tg


def test_async_snapshots_stop_at_abort(cw, ora, problems):
    """The reference throws at node 16, t = 2.04 ms: snapshots up to t = 2.0 are
    delivered, none after (the drop-in checks the failure record at each one)."""
    p = problems.c1(t_end=10.0, k0_down=1)
    setup = p.setup()
    snaps = []
    setup.snapshot_interval_ms = 0.5
    setup.on_snapshot = lambda t, v: snaps.append(t)
    with pytest.raises(cw.InstabilityError) as e:
        cw.run_simulation(p.initial_state(), setup, p.cfg)
    assert (e.value.node_index, e.value.time_ms) == (16, 2.04)
    assert [round(t, 9) for t in snaps] == [0.0, 0.5, 1.0, 1.5, 2.0]


def test_compare_schemes_one_device_operator(cw, ora, problems):
    """cli_compare (runner.cpp:254-324) on one integrator: each scheme's run,
    after cwg_set_scheme on the resident operator, equals a fresh integrator's
    run bit for bit, and the metrics are the reference's functions of them."""
    from paper_2011_04747_b200 import postprocess as pp
    p = problems.c1(model="aliev-panfilov", t_end=400.0, k0_down=1)  # long enough to repolarise (APD maps)
    p.probes = [p.sheet.nearest(0.2, 0.5), p.sheet.nearest(0.8, 0.5)]
    setup = p.setup()
    rep = pp.compare_schemes(p.initial_state(), setup, p.cfg, p.sheet.coords, reference="OST",
                             model_of_node=p.model_of_node)
    assert rep.reference == "OST" and [c.scheme for c in rep.schemes] == ["OST", "OSTAR", "DAETI"]
    for c in rep.schemes:
        sch = cw.scheme_from_string(c.scheme)
        sc = cw.SchemeConfig(scheme=sch, dt_ms=0.01 if sch == cw.Scheme.OST else 0.1, t_end_ms=400.0,
                             k0_up=p.cfg.k0_up, k0_down=p.cfg.k0_down)
        fresh = cw.run_simulation(p.initial_state(), setup, sc)
        assert np.array_equal(c.result.final_state.v, fresh.final_state.v), c.scheme
        assert np.array_equal(c.result.k_histogram, fresh.k_histogram), c.scheme
        assert np.array_equal(c.result.traces[0].v_mv, fresh.traces[0].v_mv), c.scheme
        if c.scheme == "DAETI":  # and against the oracle
            o = oracle_run(p, scheme="DAETI", dt=0.1, t_end=400.0)
            assert np.array_equal(c.result.final_state.v, o["v"])
        assert c.cv_cm_per_ms > 0 and math.isfinite(c.cv_cm_per_ms)
    ost = rep.schemes[0]
    assert ost.e_lat == 0.0 and ost.max_dv_per_probe == [0.0, 0.0]
    for c in rep.schemes[1:]:
        assert c.e_lat == pp.nrmse(ost.result.lat_map, c.result.lat_map) and 0.0 < c.e_lat < 0.5
        assert c.e_apd == pp.nrmse(ost.result.apd90_map, c.result.apd90_map)
        assert all(math.isfinite(a) for a in c.apd90_per_probe) and all(d >= 0 for d in c.max_dv_per_probe)


@pytest.mark.parametrize("model", ["aliev-panfilov", "ohara2011-epi"])
def test_generic_csr_operator_run(cw, ora, problems, model):
    """The generic CSR operator path (any mesh; diffuse_csr) through a whole run:
    bit-identical to the stencil path and to the oracle for AP, within
    tolerance for ORd."""
    from paper_2011_04747_b200 import _lib as L
    p = problems.c1(model=model, t_end=8.0, k0_down=1 if model == "aliev-panfilov" else 3)
    setup = p.setup()
    integ = cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node, op_kind=L.OP_CSR)
    try:
        r_csr = cw.run_simulation(p.initial_state(), setup, p.cfg, integrator=integ)
    finally:
        integ.close()
    r_st = gpu_run(p)
    o = oracle_run(p)
    assert np.array_equal(r_csr.final_state.v, r_st.final_state.v)
    assert np.array_equal(r_csr.k_histogram, o["k_histogram"])
    if model == "aliev-panfilov":
        assert np.array_equal(r_csr.final_state.v, o["v"])
    else:
        assert np.max(np.abs(r_csr.final_state.v - o["v"])) <= V_TOL_MV
