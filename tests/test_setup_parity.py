"""Host setup (include/cwgpu_setup.h) against the reference's own setup path:
the CSR operator, lumped mass, Gershgorin dt_s, fibrosis tags and node
selections must be bit-identical (mesh.cpp:72-180, fem.cpp:21-192)."""
import math

import numpy as np
import pytest

import paper_2011_04747_b200 as cw

GEOMS = [
    dict(lx=1.0, ly=1.0, h=0.01, ang=0.0, d0=0.001, rho=1.0),                # C1
    dict(lx=5.0, ly=5.0, h=0.025, ang=math.pi / 4, d0=0.0012, rho=0.25),    # C2
    dict(lx=2.0, ly=2.0, h=0.02, ang=0.3, d0=0.0017, rho=0.25, frac=0.25, seed=9),  # fibrotic
    dict(lx=0.5, ly=0.3, h=0.05, ang=1.1, d0=0.0013, rho=0.5),
]


@pytest.mark.parametrize("g", GEOMS)
def test_operator_bitwise(ref, g):
    frac, seed = g.get("frac", 0.0), g.get("seed", 0)
    ours = cw.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0_myocyte=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed)
    theirs = ref.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed)
    rp, col, val, mass = theirs.csr()
    assert ours.n == theirs.n
    assert np.array_equal(ours.op.row_ptr, rp)
    assert np.array_equal(ours.op.col, col)
    assert np.array_equal(ours.op.val, val)
    assert np.array_equal(ours.op.lumped_mass, mass)
    assert ours.op.dt_s == theirs.dt_s
    tags, names = theirs.tags()
    assert np.array_equal(ours.tags, tags)


def test_known_dt_s_values(ref):
    # SPEC.md:139 (5x5 cm, h = 100 um, d0 0.0017, rho 0.25): reference gives 0.0132353
    s = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.0017, rho=0.25)  # dt_s depends on h, not on the extent
    assert abs(s.op.dt_s - 0.0132353) < 1e-6
    # h^2 scaling
    a = cw.Sheet(1.0, 1.0, 0.02, 0.0).op.dt_s
    b = cw.Sheet(1.0, 1.0, 0.01, 0.0).op.dt_s
    assert abs(a / b - 4.0) < 0.05


@pytest.mark.parametrize("sel", [
    ("x_le", dict(value=0.05)), ("x_ge", dict(value=0.95)), ("y_le", dict(value=0.0)), ("y_ge", dict(value=0.5)),
    ("rectangle", dict(x0=0.2, x1=0.4, y0=0.1, y1=0.3)), ("disc", dict(cx=0.0, cy=0.0, radius=0.05)),
    ("disc", dict(cx=0.5, cy=0.5, radius=0.2)), ("node_set", dict(nodes=(5, 3, 3, 99))),
])
def test_select_nodes(ref, sel):
    ours = cw.Sheet(1.0, 1.0, 0.01, 0.0)
    theirs = ref.Sheet(1.0, 1.0, 0.01, 0.0)
    assert np.array_equal(ours.select(sel[0], **sel[1]), theirs.select(sel[0], **sel[1]))
    for x, y in [(0.5, 0.5), (0.0, 0.0), (0.333, 0.777), (1.0, 1.0)]:
        assert ours.nearest(x, y) == theirs.nearest(x, y)


def test_validation_errors():
    with pytest.raises(cw.ValidationError):
        cw.Sheet(1.0, 1.0, 0.03, 0.0)  # not a multiple of h
    with pytest.raises(cw.ValidationError):
        cw.Sheet(1.0, 1.0, 0.1, 0.0, rho=1.5)


def test_scar_extension_gershgorin_skips_zero_rows():
    ne = 20 * 20
    scale = np.ones(ne)
    scale[150:170] = 0.0
    s = cw.Sheet(1.0, 1.0, 0.05, 0.0, elem_scale=scale)
    full = cw.Sheet(1.0, 1.0, 0.05, 0.0)
    assert s.op.dt_s >= full.op.dt_s - 1e-15
    assert np.all(np.isfinite(s.op.val))
    with pytest.raises(cw.ValidationError):
        cw.Sheet(1.0, 1.0, 0.05, 0.0, elem_scale=np.zeros(ne))


def test_slab3d_tables_match_oracle_csr(ora):
    """3D extension: per-class device tables == the oracle's CSR assembly, bit for bit (incl. dt_s)."""
    import numpy as np
    sl = cw.Slab3D(0.14, 0.1, 0.08, 0.02)
    (rp, col, val, mass), dts = ora.assemble_slab3d(sl.nx, sl.ny, sl.nz, sl.h, sl.d_long, sl.rho, sl.angles)
    assert dts == sl.dt_s
    for iy in range(sl.ny1):
        for iz in range(sl.nz1):
            for ix in range(sl.nx1):
                i = int(sl.index(ix, iy, iz))
                bx = 0 if ix == 0 else (2 if ix == sl.nx else 1)
                by = 0 if iy == 0 else (2 if iy == sl.ny else 1)
                c = (by * 3 + bx) * sl.nz1 + iz
                assert mass[i] == sl.mass[c]
                present = np.zeros(27, bool)
                for p in range(rp[i], rp[i + 1]):
                    d = int(col[p] - i)
                    dy = int(round(d / sl.plane))
                    r = d - dy * sl.plane
                    dz = int(round(r / sl.nx1))
                    dx = r - dz * sl.nx1
                    q = (dy + 1) * 9 + (dz + 1) * 3 + (dx + 1)
                    present[q] = True
                    assert val[p] == sl.coef[c * 27 + q]
                assert np.all(sl.coef[c * 27:(c + 1) * 27][~present] == 0.0)
    # operator sanity: symmetric, zero row sums, lumped mass = volume
    assert abs(mass.sum() - 0.14 * 0.1 * 0.08) < 1e-15
    rs = np.add.reduceat(val, rp[:-1])
    assert np.abs(rs).max() < 1e-18


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_spectral_bound_of_gershgorin_step(which):
    """The reference's spectral-bound oracle (tests/oracles/oracles.cpp:11-60, power iteration) restated
    with a Lanczos eigensolver: lambda_max(M^-1 K) * dt_s <= 0.9 (Gershgorin discs, fem.cpp:178-192).
    C1's 0.675 puts 3 dt_s past 2, the divergence the GPU test checks (test_gpu_properties.py)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    if which == "c1":
        sh = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0)
    else:
        sh = cw.Sheet(5.0, 5.0, 0.025, math.pi / 4, d0_myocyte=0.0012, rho=0.25)
    op = sh.op
    k = sp.csr_matrix((op.val, op.col, op.row_ptr), shape=(sh.n, sh.n))
    mh = sp.diags(1.0 / np.sqrt(np.asarray(op.lumped_mass)))
    a = mh @ k @ mh
    lam = sla.eigsh((a + a.T) * 0.5, k=1, which="LA", return_eigenvectors=False)[0]
    assert 0.0 < lam * op.dt_s <= 0.9 + 1e-12
    if which == "c1":
        assert abs(lam * op.dt_s - 0.675) < 1e-9 and 3.0 * op.dt_s * lam > 2.0


@pytest.mark.parametrize("g", GEOMS)
def test_mesh_only_sheet(g):
    """cwg_sheet_mesh (the host half of the device-assembly path) builds the same coordinates and fibrosis
    tags as the full host build, and cwg_sheet2d_nnz predicts the CSR size the device assembly writes."""
    import ctypes as C
    from paper_2011_04747_b200 import _lib as L
    frac, seed = g.get("frac", 0.0), g.get("seed", 0)
    full = cw.Sheet(g["lx"], g["ly"], g["h"], g["ang"], d0_myocyte=g["d0"], rho=g["rho"], fib_fraction=frac, seed=seed)
    lib = L.lib()
    h, err = C.c_void_p(), L.cwg_error()
    assert lib.cwg_sheet_mesh(g["lx"], g["ly"], g["h"], frac, seed, C.byref(h), C.byref(err)) == 0
    try:
        n = lib.cwg_sheet_nodes(h)
        assert n == full.n and lib.cwg_sheet_nnz(h) == 0
        coords = np.ctypeslib.as_array(lib.cwg_sheet_coords(h), (n, 2))
        tags = np.ctypeslib.as_array(lib.cwg_sheet_tags(h), (n,))
        assert np.array_equal(coords, full.coords) and np.array_equal(tags, full.tags)
        d = L.cwg_sheet2d(full.nx1 - 1, full.ny1 - 1, g["h"], g["ang"], g["d0"], 0.00066, g["rho"], None, None)
        assert lib.cwg_sheet2d_nnz(C.byref(d)) == len(full.op.val)
    finally:
        lib.cwg_sheet_free(h)
