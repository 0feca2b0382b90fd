"""Golden fixtures produced by the reference itself (tests/golden/make_golden.py).

CPU part: pins the C restatement oracle against the reference's stored
outputs (so the oracle is trustworthy on a box where the reference cannot be
built). GPU part: the CUDA path against the same stored outputs.
Arithmetic-only results (Aliev-Panfilov, rules, dt_s) must match bit for bit;
libm-dependent ORd / MacCannell outputs to 1e-12 relative (glibc picks
FMA-specialised exp/log variants per host CPU).
"""
import os

import numpy as np
import pytest

from helpers import gpu_run

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODELS = ["aliev-panfilov", "ohara2011-endo", "ohara2011-epi", "ohara2011-mid", "maccannell2007"]


@pytest.fixture(scope="module")
def gold():
    return {name: np.load(os.path.join(G, name + ".npz")) for name in ("rates", "rules", "runs")}


@pytest.mark.parametrize("model", MODELS)
def test_oracle_rates_golden(ora, gold, model):
    g = gold["rates"]
    k = model.replace("-", "_")
    assert np.array_equal(ora.rest_state(model), g[k + "_rest"])
    assert ora.stable_step(model) == g[k + "_stable_step"][0]
    dv, ds = ora.rates(model, g[k + "_v"], g[k + "_s"], g[k + "_ist"])
    if model == "aliev-panfilov":
        assert np.array_equal(dv, g[k + "_dv"]) and np.array_equal(ds, g[k + "_ds"])
    else:
        np.testing.assert_allclose(dv, g[k + "_dv"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(ds, g[k + "_ds"], rtol=1e-12, atol=1e-300)


def test_oracle_rules_golden(ora, gold):
    names = ["OST", "OSTAR", "DAETI"]
    for d, sch, k0u, k0d, km, k, dt, dts, strict, l, dt_ad in gold["rules"]["rows"]:
        sch = names[int(sch)]
        assert ora.reaction_substeps(d, sch, int(k0u), int(k0d), int(km)) == int(k)
        assert ora.diffusion_substeps(dt, dts, bool(strict), sch) == (int(l), dt_ad)


def test_oracle_runs_golden(ora, gold):
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import problems
    g = gold["runs"]
    p = problems.c1(model="aliev-panfilov", t_end=40.0, k0_down=1)
    p.probes = [0, 5050, 10200]
    from helpers import oracle_run
    o = oracle_run(p)
    assert np.array_equal(o["v"], g["ap_v"])
    assert np.array_equal(o["s"], g["ap_s"])
    assert np.array_equal(o["k_histogram"], g["ap_khist"])
    assert np.array_equal(o["traces"], g["ap_traces"])
    assert np.array_equal(o["lat_valid"], g["ap_lat_valid"])
    assert np.array_equal(o["lat"][o["lat_valid"]], g["ap_lat"][g["ap_lat_valid"]])
    p = problems.c1(t_end=5.0)
    p.probes = [0, 5050, 10200]
    o = oracle_run(p)
    assert np.max(np.abs(o["v"] - g["ord_v"])) < 1e-10
    assert np.array_equal(o["k_histogram"], g["ord_khist"])
    with pytest.raises(ora.OracleInstability) as e:
        oracle_run(problems.c1(t_end=5.0, k0_down=1))
    assert (e.value.node, e.value.t) == (int(g["abort_node"][0]), float(g["abort_t"][0]))
    dts = [cw.Sheet(1, 1, 0.01, 0.0, d0_myocyte=0.001, rho=1.0).op.dt_s,
           cw.Sheet(5, 5, 0.025, np.pi / 4, d0_myocyte=0.0012, rho=0.25).op.dt_s,
           cw.Sheet(1, 1, 0.01, 0.0, d0_myocyte=0.0017, rho=0.25).op.dt_s]
    assert np.array_equal(np.array(dts), g["dt_s"])


# ----------------------------------------------------------------------------- GPU vs the same fixtures
@pytest.mark.gpu
def test_gpu_runs_golden(gold):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2011_04747_b200 import problems
    g = gold["runs"]
    p = problems.c1(model="aliev-panfilov", t_end=40.0, k0_down=1)
    p.probes = [0, 5050, 10200]
    r = gpu_run(p)
    assert np.array_equal(r.final_state.v, g["ap_v"])
    assert np.array_equal(r.k_histogram, g["ap_khist"])
    assert np.array_equal(np.array([t.v_mv for t in r.traces]), g["ap_traces"])
    assert np.array_equal(r.lat_map.value[r.lat_map.valid], g["ap_lat"][g["ap_lat_valid"]])
    p = problems.c1(t_end=5.0)
    p.probes = [0, 5050, 10200]
    r = gpu_run(p)
    assert np.max(np.abs(r.final_state.v - g["ord_v"])) < 1e-6  # north_star tolerance
    assert np.array_equal(r.k_histogram, g["ord_khist"])


@pytest.mark.gpu
@pytest.mark.parametrize("model", MODELS)
def test_gpu_rates_golden(gold, model):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    g = gold["rates"]
    k = model.replace("-", "_")
    dv, ds = cw.make_model(model).rates(g[k + "_v"], g[k + "_s"], g[k + "_ist"])
    if model == "aliev-panfilov":
        assert np.array_equal(dv, g[k + "_dv"]) and np.array_equal(ds, g[k + "_ds"])
    else:
        np.testing.assert_allclose(dv, g[k + "_dv"], rtol=1e-11, atol=1e-12)


# ----------------------------------------------------------------------------- single-cell pacing
def _pace_cases():
    src = open(os.path.join(G, "make_golden.py")).read()
    ns = {}
    exec(src[src.index("PACE_CASES ="):src.index("def pace_fixture")], ns)  # the case table only
    return ns["PACE_CASES"]


def _check_pace(model, st, mr, apd, g, i, dt, exact):
    if exact:
        assert np.array_equal(st, g[f"c{i}_state"]) and mr == g[f"c{i}_max_rel"][0]
        assert np.array_equal(apd, g[f"c{i}_apd"], equal_nan=True)
    else:  # transcendental models: libm / device exp differ by ulps; crossings are quantised to dt
        np.testing.assert_allclose(st, g[f"c{i}_state"], rtol=1e-8, atol=1e-12)
        assert abs(mr - g[f"c{i}_max_rel"][0]) < 1e-6
        ga = g[f"c{i}_apd"]
        assert np.array_equal(np.isnan(apd), np.isnan(ga))
        assert np.all(np.abs(apd[~np.isnan(ga)] - ga[~np.isnan(ga)]) <= dt * 1.0000001)


def test_oracle_pace_golden(ora):
    g = np.load(os.path.join(G, "pace.npz"))
    for i, (m, cl, nb, amp, dur) in enumerate(_pace_cases()):
        st, mr, apd = ora.pace(m, cl, nb, amp, dur)
        _check_pace(m, st, mr, apd, g, i, ora.stable_step(m) / 2, exact=(m == "aliev-panfilov"))
    with pytest.raises(ora.OracleInstability) as e:
        ora.pace("ohara2011-epi", 300.0, 2, 3000.0, 2.0)
    assert e.value.t == g["abort_t"][0]


@pytest.mark.gpu
def test_gpu_pace_golden():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    g = np.load(os.path.join(G, "pace.npz"))
    for i, (m, cl, nb, amp, dur) in enumerate(_pace_cases()):
        r = cw.pace_to_steady_state(m, cl, nb, amp, dur)
        _check_pace(m, r.state, r.max_rel_change, r.apd90_ms, g, i, cw.make_model(m).stable_step() / 2,
                    exact=(m == "aliev-panfilov"))
    with pytest.raises(cw.InstabilityError) as e:
        cw.pace_to_steady_state("ohara2011-epi", 300.0, 2, 3000.0, 2.0)
    assert e.value.time_ms == g["abort_t"][0] and e.value.node_index == -1
