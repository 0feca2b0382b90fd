"""Pin the C restatement oracle against the reference itself (oracle/_ref/libcwref.so).

Both run on this host's libm, so every comparison is bit-exact: rates() of
all five registry models, the adaptation rules (incl. SPEC.md's worked
examples), diffusion_substep, and full run_simulation outputs (final state,
k-histogram, traces, LAT/APD maps) including the reference's own abort.
"""
import math

import numpy as np
import pytest

MODELS = ["aliev-panfilov", "ohara2011-endo", "ohara2011-epi", "ohara2011-mid", "maccannell2007"]


@pytest.mark.parametrize("model", MODELS)
def test_rates_bitwise(ref, ora, model):
    rng = np.random.default_rng(7)
    ns, ss, rest = ref.model_info(model)
    assert ns == ora.state_count(model) and ss == ora.stable_step(model)
    assert np.array_equal(rest, ora.rest_state(model))
    n = 3000
    if model == "aliev-panfilov":
        v = rng.uniform(-85, 25, n)
        s = rng.uniform(0, 2, (n, 1))
    else:
        v = rng.uniform(-100, 60, n)
        s = np.tile(rest[1:], (n, 1)) * rng.uniform(0.5, 1.5, (n, ns))
    # include the x/expm1 branch point and exact rest states
    v[:3] = [0.0, 1e-9, rest[0]]
    s[2] = rest[1:]
    ist = rng.choice([0.0, 37.5, 592.0], n)
    a = ref.rates(model, v, s, ist)
    b = ora.rates(model, v, s, ist)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_spec_rule_examples(ref, ora):
    # SPEC.md:257-259 (dt 0.1, dt0 0.01 -> k_max 10; k0 5/1)
    for dvdt, k in [(120.0, 10), (-0.8, 1), (0.2, 5)]:
        assert ora.reaction_substeps(dvdt, "DAETI", 5, 1, 10) == k == ref.reaction_substeps(dvdt, "DAETI", 5, 1, 10)
    # SPEC.md:266-268
    assert ora.diffusion_substeps(0.1, 0.013, False, "DAETI") == (3, 0.1 / 6.0)
    assert ora.diffusion_substeps(0.1, 0.113, False, "DAETI") == (1, 0.05)
    assert ora.diffusion_substeps(0.1, 0.05, False, "DAETI") == (1, 0.05)
    assert ora.k_max_for(0.1, "ohara2011-epi") == 10 == ref.k_max_for(0.1, "ohara2011-epi")


def test_rules_random_bitwise(ref, ora):
    rng = np.random.default_rng(3)
    for _ in range(3000):
        d = float(rng.choice([-1, 1]) * 10 ** rng.uniform(-3, 3))
        sch = ["OST", "OSTAR", "DAETI"][int(rng.integers(3))]
        k0d = int(rng.integers(1, 4))
        k0u = k0d + int(rng.integers(0, 5))
        km = int(rng.integers(1, 20))
        assert ora.reaction_substeps(d, sch, k0u, k0d, km) == ref.reaction_substeps(d, sch, k0u, k0d, km)
        dt = float(rng.uniform(0.005, 0.5))
        dts = float(rng.uniform(0.001, 0.3))
        strict = bool(rng.integers(2))
        assert ora.diffusion_substeps(dt, dts, strict, sch) == ref.diffusion_substeps(dt, dts, strict, sch)


@pytest.mark.parametrize("geom", [(1, 1, 0.01, 0.0, 0.001, 1.0), (2, 1.5, 0.025, 0.7, 0.0012, 0.25)])
def test_diffusion_substep_bitwise(ref, ora, geom):
    lx, ly, h, ang, d0, rho = geom
    s = ref.Sheet(lx, ly, h, ang, d0=d0, rho=rho)
    v = np.random.default_rng(1).uniform(-90, 40, s.n)
    assert np.array_equal(s.diffusion_substep(v, 0.0123), ora.diffusion_substep(s.csr(), v, 0.0123))


def _both(ref, ora, model, sel, amp, t_end, k0_down, scheme="DAETI", dt=0.1, probes=(0, 5050, 10200)):
    s = ref.Sheet(1, 1, 0.01, 0.0, d0=0.001, rho=1.0)
    nodes = s.select(*sel[0], **sel[1])
    s.set_models([model])
    s.add_stimulus(nodes, 0.0, 1.0, amp)
    s.init_state()
    try:
        r = s.run(scheme=scheme, dt=dt, t_end=t_end, k0_down=k0_down, probes=probes)
        rerr = None
    except ref.RefError as e:
        r, rerr = None, (e.node, e.t)
    try:
        o = ora.run_simulation(s.csr(), s.dt_s, [model], np.zeros(s.n, np.uint8), [(nodes, 0.0, 1.0, amp, None)],
                               scheme=scheme, dt=dt, t_end=t_end, k0_down=k0_down, probes=probes)
        oerr = None
    except ora.OracleInstability as e:
        o, oerr = None, (e.node, e.t)
    return r, rerr, o, oerr


def test_run_ap_bitwise(ref, ora):
    r, _, o, _ = _both(ref, ora, "aliev-panfilov", (("x_le",), dict(value=0.05)), 100.0, 60.0, 1)
    assert np.array_equal(r["state"][0], o["v"])
    assert np.array_equal(r["state"][1], o["s"])
    assert np.array_equal(r["state"][2], o["last_dvdt"])
    assert np.array_equal(r["k_histogram"], o["k_histogram"])
    assert np.array_equal(np.array([tv[1] for tv in r["traces"]]), o["traces"])
    assert np.array_equal(r["lat_valid"], o["lat_valid"])
    assert np.array_equal(r["lat"][r["lat_valid"]], o["lat"][o["lat_valid"]])


def test_run_ord_bitwise(ref, ora):
    r, _, o, _ = _both(ref, ora, "ohara2011-epi", (("x_le",), dict(value=0.0)), 592.0, 6.0, 3)
    assert np.array_equal(r["state"][0], o["v"])
    assert np.array_equal(r["state"][1], o["s"])
    assert np.array_equal(r["k_histogram"], o["k_histogram"])
    assert np.array_equal(np.array([tv[1] for tv in r["traces"]]), o["traces"])


def test_abort_fixture(ref, ora):
    """ORd-epi, paper k0, 592 mV/ms -> InstabilityError at node 16, t = 2.04 ms."""
    _, rerr, _, oerr = _both(ref, ora, "ohara2011-epi", (("x_le",), dict(value=0.0)), 592.0, 5.0, 1)
    assert rerr is not None and rerr == oerr
    assert rerr[0] == 16 and abs(rerr[1] - 2.04) < 1e-12
