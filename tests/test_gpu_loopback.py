"""The multi-GPU decomposition on one device.

N slab contexts (world = N, rank r) run in loopback mode: no NCCL, the halo
rows/planes are copied between the ranks' V buffers before every diffusion
sub-step exactly where halo_exchange's ncclSend/ncclRecv would
(cwg_loopback_steps). The slab kernels, node offsets, model bins and
recording run as on N GPUs; the gathered final state must equal the
single-context run bit for bit."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    old = os.environ.get("CWG_LOOPBACK")
    os.environ["CWG_LOOPBACK"] = "1"
    yield
    if old is None:
        os.environ.pop("CWG_LOOPBACK", None)
    else:
        os.environ["CWG_LOOPBACK"] = old


def _loopback(p, world, link=False):
    """link=True: the peer-memory transport (cwg_loopback_link) instead of the NCCL-equivalent copies."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import _lib as L
    setup = p.setup()
    integs = [cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node, rank=r, world=world)
              for r in range(world)]
    try:
        st = p.initial_state()
        hs = (C.c_void_p * world)(*[it._h.value for it in integs])
        if link:
            assert L.lib().cwg_loopback_link(hs, world) == 0, L.lib().cwg_last_error().decode()
        for it in integs:
            it.upload(st)
            it.run_begin()
        n = integs[0].info.n_steps
        rc = L.lib().cwg_loopback_steps(hs, world, 0, n)
        assert rc == 0, L.lib().cwg_last_error().decode()
        out = p.initial_state()
        for it in integs:
            it.download(out)
        kh = sum(it.k_histogram() for it in integs)
        return out, kh
    finally:
        for it in integs:
            it.close()


def _single(p):
    import paper_2011_04747_b200 as cw
    os.environ["CWG_LOOPBACK"] = "0"
    try:
        return cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
    finally:
        os.environ["CWG_LOOPBACK"] = "1"


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_2d_aliev_panfilov(world):
    from paper_2011_04747_b200 import problems
    p = problems.c1(model="aliev-panfilov", t_end=15.0, k0_down=1)
    out, kh = _loopback(p, world)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v)
    assert np.array_equal(out.s, ref.final_state.s)
    assert np.array_equal(kh, ref.k_histogram)


def test_loopback_2d_ord_and_fibrosis():
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import api, problems
    p = problems.c1(t_end=4.0)
    out, kh = _loopback(p, 2)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v) and np.array_equal(kh, ref.k_histogram)
    sh = cw.Sheet(1.0, 0.5, 0.02, 0.3, d0_myocyte=0.0017, d0_fibrotic=0.00066, rho=0.25, fib_fraction=0.2, seed=5)
    nodes = sh.select("x_le", value=0.05)
    q = problems.Problem("fib", sh, ["ohara2011-epi", "maccannell2007"], sh.tags.astype(np.uint8),
                         [(nodes, 0.0, 1.0, 80.0, None)], api.SchemeConfig(dt_ms=0.1, t_end_ms=3.0, k0_down=3), [0])
    out, kh = _loopback(q, 3)
    ref = _single(q)
    assert np.array_equal(out.v, ref.final_state.v) and np.array_equal(kh, ref.k_histogram)


def test_loopback_3d_slab():
    from paper_2011_04747_b200 import problems
    p = problems.slab(0.4, 0.3, 0.2, 0.02, model="aliev-panfilov", t_end=10.0, amplitude=100.0)
    out, kh = _loopback(p, 2)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v)
    assert np.array_equal(kh, ref.k_histogram)


def test_loopback_thin_slabs():
    """Slabs of 2-3 rows with several diffusion sub-steps per step: every
    sub-step's halo row is exchanged; still bit-identical."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import api, problems
    sh = cw.Sheet(1.0, 0.1, 0.02, 0.3, d0_myocyte=0.0017, rho=0.25)  # 6 rows
    nodes = sh.select("x_le", value=0.05)
    p = problems.Problem("thin", sh, ["aliev-panfilov"], np.zeros(sh.n, np.uint8), [(nodes, 0.0, 1.0, 100.0, None)],
                         api.SchemeConfig(dt_ms=0.3, t_end_ms=6.0), [0])
    assert cw.diffusion_substeps(0.3, sh.op.dt_s, False, cw.Scheme.DAETI).l >= 2
    for world in (2, 3):  # 3 and 2 rows per rank
        out, kh = _loopback(p, world)
        ref = _single(p)
        assert np.array_equal(out.v, ref.final_state.v), world
        assert np.array_equal(kh, ref.k_histogram)


def test_loopback_c2_single_substep_launches():
    """C2 geometry: l = 1, so step I is a single plain-kernel sub-step and the
    merged steps are one fused launch of 2 -- both with the multi-rank halo
    offsets."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import problems
    p = problems.c2(t_end=3.0)
    assert cw.diffusion_substeps(0.1, p.sheet.op.dt_s, False, cw.Scheme.DAETI).l == 1
    out, kh = _loopback(p, 2)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v) and np.array_equal(kh, ref.k_histogram)


def _loopback_full(p, world, link=False):
    """Loopback run that also assembles the global traces (each probe recorded by its owning rank) and the
    LAT/APD maps (each rank's y-slab rows) like cwg_gather_result does over NCCL."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import _lib as L
    setup = p.setup()
    integs = [cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node, rank=r, world=world)
              for r in range(world)]
    try:
        st = p.initial_state()
        hs = (C.c_void_p * world)(*[it._h.value for it in integs])
        if link:
            assert L.lib().cwg_loopback_link(hs, world) == 0, L.lib().cwg_last_error().decode()
        for it in integs:
            it.upload(st)
            it.run_begin()
        n = integs[0].info.n_steps
        rc = L.lib().cwg_loopback_steps(hs, world, 0, n)
        assert rc == 0, L.lib().cwg_last_error().decode()
        out = p.initial_state()
        lat, lv = np.zeros(p.n), np.zeros(p.n, bool)
        apd, av = np.zeros(p.n), np.zeros(p.n, bool)
        traces = None
        plane = p.n // p.sheet.op.ny1
        for r, it in enumerate(integs):
            it.download(out)
            rb, re = cw.slab_plan(p.sheet.op.ny1, world, r)
            lm, am = it.maps()
            lat[rb * plane:re * plane], lv[rb * plane:re * plane] = lm.value, lm.valid
            apd[rb * plane:re * plane], av[rb * plane:re * plane] = am.value, am.valid
            _, tv = it.traces()
            traces = tv if traces is None else traces + tv  # a probe's non-owning ranks record 0
        kh = sum(it.k_histogram() for it in integs)
        return out, kh, traces, (lat, lv), (apd, av)
    finally:
        for it in integs:
            it.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_loopback_c4_geometry_traces_and_maps(world):
    """BASELINE configs[3] at full size (251 x 251 x 51) split into 2 / 4 / 8 y-slabs: state, k-histogram,
    probe traces and LAT/APD maps bit-identical to the single-context run (the multi-GPU analogue of the
    reference's worker-count determinism)."""
    from paper_2011_04747_b200 import problems
    p = problems.c4(t_end=8.0)
    out, kh, tr, (lat, lv), (apd, av) = _loopback_full(p, world)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v)
    assert np.array_equal(out.s, ref.final_state.s)
    assert np.array_equal(kh, ref.k_histogram)
    assert np.array_equal(tr, np.array([t.v_mv for t in ref.traces]))
    assert np.array_equal(lv, ref.lat_map.valid) and np.array_equal(lat[lv], ref.lat_map.value[lv])
    assert np.array_equal(av, ref.apd90_map.valid) and np.array_equal(apd[av], ref.apd90_map.value[av])
    assert lv.sum() > 0  # the endocardial wave has activated nodes within the window


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_memory_transport_c4(world):
    """The peer-memory (P2P) transport's data path on the full C4 grid: linked rank contexts store the
    neighbours' halo planes from inside the diffusion kernel (and push them after the reaction), pacing on
    launch counters -- bit-identical to one context."""
    from paper_2011_04747_b200 import problems
    p = problems.c4(t_end=6.0)
    out, kh, tr, (lat, lv), (apd, av) = _loopback_full(p, world, link=True)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v)
    assert np.array_equal(out.s, ref.final_state.s)
    assert np.array_equal(kh, ref.k_histogram)
    assert np.array_equal(tr, np.array([t.v_mv for t in ref.traces]))
    assert np.array_equal(lv, ref.lat_map.valid) and np.array_equal(lat[lv], ref.lat_map.value[lv])


@pytest.mark.parametrize("world", [2, 3])
def test_peer_memory_transport_2d(world):
    """2D: fused diffusion launches (T <= H halo rows) store H halo rows into the neighbours; ORd C2 sheet
    (l = 1: the merged step is one fused launch of 2) and the thin-slab AP case (several launches per step)."""
    from paper_2011_04747_b200 import problems
    p = problems.c2(t_end=3.0)
    out, kh = _loopback(p, world, link=True)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v) and np.array_equal(kh, ref.k_histogram)
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import api
    sh = cw.Sheet(1.0, 0.6, 0.02, 0.3, d0_myocyte=0.0017, rho=0.25)  # 31 rows: >= 2 H per rank
    nodes = sh.select("x_le", value=0.05)
    q = problems.Problem("thin", sh, ["aliev-panfilov"], np.zeros(sh.n, np.uint8), [(nodes, 0.0, 1.0, 100.0, None)],
                         api.SchemeConfig(dt_ms=0.3, t_end_ms=6.0), [0])
    out, kh = _loopback(q, world, link=True)
    ref = _single(q)
    assert np.array_equal(out.v, ref.final_state.v) and np.array_equal(kh, ref.k_histogram)


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_c3_tma_slabs(world):
    """BASELINE configs[2] (C3, 1001 x 1001, 22 diffusion sub-steps per step) in y-slabs: the TMA-fed register-quad
    diffusion kernel runs on the slabs too (coefficient tensor with the halo rows, fused depth <= the halo depth,
    exchanges between launches) -- bit-identical to the single context, which fuses up to 6 sub-steps."""
    from paper_2011_04747_b200 import problems
    p = problems.c3(t_end=2.0)
    out, kh = _loopback(p, world)
    ref = _single(p)
    assert np.array_equal(out.v, ref.final_state.v)
    assert np.array_equal(out.s, ref.final_state.s)
    assert np.array_equal(kh, ref.k_histogram)
