"""Edge cases of the hot path on the CUDA side, each against the CPU oracle.

Degenerate and ragged geometries (a single element, one-element-wide strips,
a 1-row-of-elements sheet), the shortest runs (one outer step: step I, A and
III at once, splitting.cpp:171-181), runs without a stimulus or without
probes, and a stimulus that is still on when the run ends. Aliev-Panfilov
cases are bit-exact; ORd ones are held to the 1e-6 mV contract.
"""
import math

import numpy as np
import pytest

from helpers import gpu_run, oracle_run

pytestmark = pytest.mark.gpu
V_TOL_MV = 1e-6


@pytest.fixture(scope="module")
def cw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    return cw


def _problem(cw, lx, ly, h, model="aliev-panfilov", t_end=5.0, dt=0.1, stim=True, probes=True, amp=100.0,
             dur=1.0, ang=0.3, k0_down=3):
    from paper_2011_04747_b200 import api, problems
    sh = cw.Sheet(lx, ly, h, ang, d0_myocyte=0.0012, rho=0.25)
    stims = [(sh.select("x_le", value=0.0), 0.0, dur, amp, None)] if stim else []
    pr = [0, sh.n - 1] if probes else []
    return problems.Problem("edge", sh, [model], np.zeros(sh.n, np.uint8), stims,
                            api.SchemeConfig(dt_ms=dt, t_end_ms=t_end, k0_down=k0_down), pr)


def _exact(res, o):
    assert np.array_equal(res.final_state.v, o["v"])
    assert np.array_equal(res.final_state.s.reshape(o["s"].shape), o["s"])
    assert np.array_equal(res.k_histogram, o["k_histogram"])
    for q, tr in enumerate(res.traces):
        assert np.array_equal(tr.v_mv, o["traces"][q])
    assert np.array_equal(res.lat_map.valid, o["lat_valid"])
    assert np.array_equal(res.lat_map.value[o["lat_valid"]], o["lat"][o["lat_valid"]])


@pytest.mark.parametrize("lx,ly,h", [(0.02, 0.02, 0.02),    # one element, 4 nodes
                                     (0.02, 0.5, 0.02),     # a strip one element wide in x
                                     (0.5, 0.02, 0.02),     # one row of elements
                                     (0.07, 0.13, 0.01)])   # ragged 8 x 14 nodes
def test_degenerate_and_ragged_sheets_bitwise(cw, lx, ly, h):
    p = _problem(cw, lx, ly, h, t_end=8.0)
    _exact(gpu_run(p), oracle_run(p))


@pytest.mark.parametrize("t_end", [0.1, 0.2])  # one step (I + A + III), two steps (I + A + B, then A + III)
def test_shortest_runs_bitwise(cw, t_end):
    p = _problem(cw, 0.3, 0.2, 0.01, t_end=t_end)
    _exact(gpu_run(p), oracle_run(p))


def test_no_stimulus_no_probes_bitwise(cw):
    p = _problem(cw, 0.3, 0.2, 0.01, stim=False, probes=False, t_end=3.0)
    res, o = gpu_run(p), oracle_run(p)
    _exact(res, o)
    assert not res.lat_map.valid.any()  # nothing activates


def test_stimulus_on_at_the_end_ord(cw):
    """ORd, the stimulus window still open when the run stops (t_end inside [t0, t0 + dur))."""
    p = _problem(cw, 0.3, 0.3, 0.02, model="ohara2011-epi", t_end=1.5, dur=5.0, amp=80.0)
    res, o = gpu_run(p), oracle_run(p)
    assert np.max(np.abs(res.final_state.v - o["v"])) <= V_TOL_MV
    assert np.array_equal(res.k_histogram, o["k_histogram"])
    for q, tr in enumerate(res.traces):
        assert np.max(np.abs(tr.v_mv - o["traces"][q])) <= V_TOL_MV


@pytest.mark.parametrize("lx,ly,lz", [(0.02, 0.12, 0.02),   # one element in x and z
                                      (0.3, 0.02, 0.04),    # one element in y (the slab axis)
                                      (0.06, 0.1, 0.02)])   # one element layer in z (fibre angle +60 only)
def test_degenerate_3d_slabs_bitwise(cw, lx, ly, lz):
    from paper_2011_04747_b200 import problems
    p = problems.slab(lx, ly, lz, 0.02, model="aliev-panfilov", t_end=6.0, amplitude=100.0)
    _exact(gpu_run(p), oracle_run(p))


@pytest.mark.parametrize("model", ["ohara2011-endo", "ohara2011-mid", "maccannell2007"])
def test_other_cell_models_full_runs(cw, model):
    """Whole DAETI runs of the other registered models (ohara_rudy_2011.cpp:86-87 cell types,
    maccannell_2007.cpp) on the C1 sheet -- the tolerance contract, identical k-histograms."""
    from paper_2011_04747_b200 import problems
    p = problems.c1(model=model, t_end=12.0, amplitude=600.0 if model != "maccannell2007" else 100.0)
    res, o = gpu_run(p), oracle_run(p)
    assert np.max(np.abs(res.final_state.v - o["v"])) <= V_TOL_MV
    assert np.array_equal(res.k_histogram, o["k_histogram"])
    for q, tr in enumerate(res.traces):
        assert np.max(np.abs(tr.v_mv - o["traces"][q])) <= V_TOL_MV


@pytest.mark.parametrize("scheme,dt,strict", [("OSTAR", 0.1, False), ("DAETI", 0.1, True), ("OST", 0.02, False)])
def test_ord_schemes_and_strict_substeps(cw, scheme, dt, strict):
    """ORd under the other schemes and the strict (ceil) diffusion sub-step rule (splitting.cpp:56-67)."""
    from paper_2011_04747_b200 import api, problems
    p = problems.c1(t_end=8.0, scheme=api.Scheme[scheme], dt=dt)
    p.cfg.strict_substeps = strict
    res, o = gpu_run(p), oracle_run(p)
    assert np.max(np.abs(res.final_state.v - o["v"])) <= V_TOL_MV
    assert np.array_equal(res.k_histogram, o["k_histogram"])


def test_record_interval_not_a_multiple_of_dt(cw):
    """Traces every llround(rec / dt) steps (splitting.cpp:274-279) with rec = 0.35 ms at dt = 0.1 (AP, bit-exact)."""
    p = _problem(cw, 0.3, 0.2, 0.01, t_end=6.0)
    p.cfg.record_interval_ms = 0.35
    res, o = gpu_run(p), oracle_run(p)
    _exact(res, o)
    assert len(res.traces[0].v_mv) == len(o["traces"][0])


def test_3d_kernels_agree():
    """The register-blocked 3D diffusion kernel (default) and the round-1 shared-memory ring kernel
    (CWG_S3_KERNEL=0) give the same bits on an ORd slab with every node class (faces, edges, corners)."""
    import os
    from paper_2011_04747_b200 import problems
    from helpers import gpu_run
    p = problems.slab(0.6, 0.5, 0.3, 0.02, t_end=3.0)
    old = os.environ.get("CWG_S3_KERNEL")
    try:
        os.environ["CWG_S3_KERNEL"] = "0"
        a = gpu_run(p)
    finally:
        if old is None:
            os.environ.pop("CWG_S3_KERNEL", None)
        else:
            os.environ["CWG_S3_KERNEL"] = old
    b = gpu_run(p)
    assert np.array_equal(a.final_state.v, b.final_state.v)
    assert np.array_equal(a.final_state.s, b.final_state.s)
    assert np.array_equal(a.k_histogram, b.k_histogram)


@pytest.mark.parametrize("models,extra", [(["ohara2011-epi"], 0), (["aliev-panfilov"], 0), (["maccannell2007"], 3),
                                          (["ohara2011-endo", "maccannell2007"], 5), (["aliev-panfilov"], 2)])
def test_state_upload_download_round_trip(cw, models, extra):
    """The device keeps the states column-wise in groups of four (common.cuh sidx, 32-byte refill accesses);
    whatever the model's state count (40, 2, 1: full groups and ragged tails) and the caller's stride (>= the
    largest state count, e.g. a checkpoint of a wider model list), upload then download returns the caller's
    NodeStateArray bit for bit in the columns the models own and zeros beyond (ionic.hpp:39-55)."""
    from paper_2011_04747_b200 import api, problems
    sh = cw.Sheet(0.21, 0.13, 0.01, 0.3, d0_myocyte=0.0012, rho=0.25)
    rng = np.random.default_rng(7)
    mon = (np.arange(sh.n) % len(models)).astype(np.uint8)
    p = problems.Problem("layout", sh, models, mon, [], api.SchemeConfig(dt_ms=0.1, t_end_ms=1.0, k0_down=3), [])
    integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=mon)
    try:
        st0 = p.initial_state()
        stride = st0.stride + extra
        counts = np.array([cw.make_model(m).state_count() for m in models])[mon]
        s = rng.standard_normal((sh.n, stride))
        s[np.arange(stride)[None, :] >= counts[:, None]] = 0.0
        st = api.NodeStateArray(sh.n, stride, rng.standard_normal(sh.n), s.reshape(-1).copy(),
                                rng.standard_normal(sh.n), mon)
        integ.upload(st)
        back = api.NodeStateArray(sh.n, stride, np.full(sh.n, np.nan), np.full(sh.n * stride, np.nan),
                                  np.full(sh.n, np.nan), mon)
        integ.download(back)
        assert np.array_equal(back.v, st.v)
        assert np.array_equal(back.last_dvdt, st.last_dvdt)
        assert np.array_equal(back.s, st.s)
    finally:
        integ.close()
