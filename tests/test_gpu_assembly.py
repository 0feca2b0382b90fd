"""Device assembly of regular sheets (assemble.cu, cwg_sheet2d_assemble,
CWG_OP_SHEET2D) against the reference's assemble + gershgorin_step (fem.cpp:21-192).

Contract: the CSR structure, the lumped mass and every off-diagonal entry
are bit-identical to the reference's; a diagonal entry sums its four element contributions in
ascending element order, the reference in std::sort's tie order (fem.cpp:135-145), so it may differ by
at most 2 ulp; dt_s likewise. Runs on a device-assembled operator stay within the ORd tolerance of the
host-assembled ones."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GEOMS = [
    dict(lx=1.0, ly=1.0, h=0.01, ang=0.0, d0=0.001, rho=1.0),                # C1
    dict(lx=5.0, ly=5.0, h=0.025, ang=math.pi / 4, d0=0.0012, rho=0.25),    # C2
    dict(lx=2.0, ly=2.0, h=0.02, ang=0.3, d0=0.0017, rho=0.25, frac=0.25, seed=9),  # fibrotic
    dict(lx=0.5, ly=0.3, h=0.05, ang=1.1, d0=0.0013, rho=0.5),
]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ulps(a, b):
    return np.abs(a.view(np.int64) - b.view(np.int64))


def _compare(dev, host):
    """dev / host AssembledOperator: structure and mass equal, off-diagonals bitwise, diagonals <= 2 ulp."""
    assert np.array_equal(dev.row_ptr, host.row_ptr)
    assert np.array_equal(dev.col, host.col)
    assert np.array_equal(dev.lumped_mass.view(np.int64), host.lumped_mass.view(np.int64))
    rows = np.repeat(np.arange(len(host.lumped_mass)), np.diff(host.row_ptr))
    diag = host.col == rows
    assert np.array_equal(dev.val[~diag].view(np.int64), host.val[~diag].view(np.int64))
    u = _ulps(dev.val[diag], host.val[diag])
    assert u.max() <= 2
    assert _ulps(np.array([dev.dt_s]), np.array([host.dt_s]))[0] <= 2
    return int((u > 0).sum()), int(diag.sum())


@pytest.mark.parametrize("g", GEOMS)
def test_device_csr_vs_host(g):
    import paper_2011_04747_b200 as cw
    frac, seed = g.get("frac", 0.0), g.get("seed", 0)
    host = cw.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0_myocyte=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed)
    dev = cw.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0_myocyte=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed,
                   assembly="device")
    assert np.array_equal(dev.coords, host.coords) and np.array_equal(dev.tags, host.tags)
    _compare(dev.op.csr(), host.op)


@pytest.mark.parametrize("g", GEOMS[:3])
def test_device_csr_vs_reference(ref, g):
    """Directly against the unmodified reference's assemble (oracle/_ref/libcwref.so)."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200.api import AssembledOperator
    frac, seed = g.get("frac", 0.0), g.get("seed", 0)
    theirs = ref.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed)
    rp, col, val, mass = theirs.csr()
    dev = cw.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0_myocyte=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed,
                   assembly="device")
    differ, total = _compare(dev.op.csr(), AssembledOperator(rp, col, val, mass, theirs.dt_s))
    assert differ < total  # most diagonals agree bit for bit too


def test_device_csr_c3_scar():
    """BASELINE configs[2] (C3) at full size: 1001^2 nodes with the scar (D = 0 elements) and border zone;
    Gershgorin skips the scar's zero rows like the host path."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import problems
    host = problems.c3().sheet
    h, size = 0.005, 5.0
    nx = int(round(size / h))
    ex = (np.arange(nx) + 0.5) * h
    X, Y = np.meshgrid(ex, ex)
    r = np.hypot(X - size / 2, Y - size / 2).ravel()
    scale = np.where(r <= 1.0, 0.0, np.where(r <= 1.5, 0.5, 1.0))
    dev = cw.Sheet(size, size, h, 0.0, d0_myocyte=0.001, rho=1.0, elem_scale=scale, assembly="device")
    differ, total = _compare(dev.op.csr(), host.op)
    assert total == host.n


@pytest.mark.parametrize("bad,msg", [
    (dict(rho=0.0), "diffusion: rho must lie in (0, 1]"),
    (dict(d0_myocyte=-1.0), "diffusion: coefficients must be positive"),
])
def test_device_assembly_validation(bad, msg):
    import paper_2011_04747_b200 as cw
    kw = dict(d0_myocyte=0.001, rho=1.0)
    kw.update(bad)
    with pytest.raises(cw.ValidationError) as e_dev:
        cw.Sheet(1.0, 1.0, 0.05, 0.0, assembly="device", **kw)
    with pytest.raises(cw.ValidationError) as e_host:
        cw.Sheet(1.0, 1.0, 0.05, 0.0, **kw)
    assert str(e_dev.value) == str(e_host.value) == msg


def _run(sheet, model, t_end, world=1):
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import api, problems
    nodes = sheet.select("x_le", value=0.05)
    amp = 100.0  # x <= 0.05 strip: stable for ORd-epi at k0_down = 3 (SURVEY.md §8d C2 caution 2)
    p = problems.Problem("asm", sheet, [model], np.zeros(sheet.n, np.uint8), [(nodes, 0.0, 1.0, amp, None)],
                         api.SchemeConfig(dt_ms=0.1, t_end_ms=t_end, k0_up=5, k0_down=3), [sheet.nearest(0.5, 0.5)])
    return cw.run_simulation(p.initial_state(), p.setup(), p.cfg), p


@pytest.mark.parametrize("model", ["aliev-panfilov", "ohara2011-epi"])
def test_run_on_device_operator(model):
    """C1 geometry: a run on the device-assembled operator (CWG_OP_SHEET2D) against the same run on the
    host-assembled one -- identical plan, k-histogram and LAT validity, V within the ORd tolerance."""
    import paper_2011_04747_b200 as cw
    host = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0)
    dev = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0, assembly="device")
    rh, _ = _run(host, model, 20.0)
    rd, _ = _run(dev, model, 20.0)
    assert rd.plan == rh.plan
    assert np.array_equal(rd.k_histogram, rh.k_histogram)
    assert np.max(np.abs(rd.final_state.v - rh.final_state.v)) <= 1e-6
    assert np.array_equal(rd.lat_map.valid, rh.lat_map.valid)
    assert np.max(np.abs(rd.lat_map.value[rd.lat_map.valid] - rh.lat_map.value[rh.lat_map.valid])) <= 1e-6


def test_run_on_device_operator_matches_its_csr():
    """The device-assembled stencil tables are exactly the CSR cwg_sheet2d_assemble returns: a run on
    CWG_OP_SHEET2D equals, bit for bit, the run on that CSR handed over as a host operator."""
    import paper_2011_04747_b200 as cw
    dev = cw.Sheet(2.0, 1.0, 0.02, 0.7, d0_myocyte=0.0012, rho=0.25, assembly="device")
    via_csr = cw.Sheet(2.0, 1.0, 0.02, 0.7, d0_myocyte=0.0012, rho=0.25, assembly="device")
    via_csr.op = dev.op.csr()
    ra, _ = _run(dev, "aliev-panfilov", 10.0)
    rb, _ = _run(via_csr, "aliev-panfilov", 10.0)
    assert np.array_equal(ra.final_state.v, rb.final_state.v)
    assert np.array_equal(ra.k_histogram, rb.k_histogram)


@pytest.mark.parametrize("world", [2, 3])
def test_device_operator_slabs(world):
    """y-slab contexts (loopback) slice their coefficient rows out of the device-assembled table: bit-identical
    to the single context."""
    import ctypes as C
    import os
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import _lib as L
    dev = cw.Sheet(1.0, 1.0, 0.02, 0.4, d0_myocyte=0.0012, rho=0.25, assembly="device")
    ref, p = _run(dev, "aliev-panfilov", 8.0)
    old = os.environ.get("CWG_LOOPBACK")
    os.environ["CWG_LOOPBACK"] = "1"
    try:
        setup = p.setup()
        integs = [cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node, rank=r, world=world)
                  for r in range(world)]
        hs = (C.c_void_p * world)(*[it._h.value for it in integs])
        st = p.initial_state()
        for it in integs:
            it.upload(st)
            it.run_begin()
        assert L.lib().cwg_loopback_steps(hs, world, 0, integs[0].info.n_steps) == 0, L.lib().cwg_last_error()
        out = p.initial_state()
        for it in integs:
            it.download(out)
        for it in integs:
            it.close()
    finally:
        if old is None:
            os.environ.pop("CWG_LOOPBACK", None)
        else:
            os.environ["CWG_LOOPBACK"] = old
    assert np.array_equal(out.v, ref.final_state.v)


def test_device_operator_serves_csr_entry_points():
    """The CSR-taking entry points (diffusion_substep, fem.cpp:194-207) accept a device-assembled operator: its
    CSR views are assembled once on demand, and the sub-step equals the one on .csr()."""
    import paper_2011_04747_b200 as cw
    dev = cw.Sheet(1.0, 1.0, 0.02, 0.3, d0_myocyte=0.0012, rho=0.25, assembly="device")
    v = np.random.default_rng(5).uniform(-90.0, 40.0, dev.n)
    a = cw.diffusion_substep(dev.op, v, dev.op.dt_s)
    b = cw.diffusion_substep(dev.op.csr(), v, dev.op.dt_s)
    assert np.array_equal(a, b)
    assert dev.op.entry(0, 0) == dev.op.csr().entry(0, 0)
