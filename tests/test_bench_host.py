"""Host-side checks of bench.py (CPU): the reference arm restates the problem constants and builds its
C4/C5 problems from the oracle alone (no product import), so those restatements must equal the product's
problem definitions (paper_2011_04747_b200/problems.py) and the oracle's structured slab operator must
equal its own CSR assembly."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_constants_match_problems():
    import bench
    from paper_2011_04747_b200 import problems
    assert bench.C1_AMPLITUDE == problems.C1_AMPLITUDE
    assert bench.C2_AMPLITUDE == problems.C2_AMPLITUDE
    assert bench.C2_RADIUS == problems.C2_RADIUS
    p = problems.c4(t_end=1.0)
    assert p.stimuli[0][3] == bench.SLAB_AMPLITUDE
    assert (bench.C5_AMPLITUDE, bench.C5_SITE_RADIUS) == (problems.C5_AMPLITUDE, problems.C5_SITE_RADIUS)


def test_oracle_c4_matches_product_c4():
    import bench
    from paper_2011_04747_b200 import problems
    op, nodes, t_end = bench.oracle_slab("c4")
    p = problems.c4()
    assert op.n == p.n and t_end == p.cfg.t_end_ms
    assert np.array_equal(np.sort(np.asarray(p.stimuli[0][0], np.int64)), nodes)
    assert np.array_equal(op.angles, p.sheet.op.angles)
    assert op.dt_s == p.sheet.op.dt_s  # oracle's class tables vs the product's structured tables (same Gershgorin)
    assert np.array_equal(op.coef, p.sheet.op.coef) and np.array_equal(op.mass, p.sheet.op.mass)


def test_oracle_c5_sites_match_product():
    import bench
    from paper_2011_04747_b200 import problems
    op, nodes, _ = bench.oracle_slab("c5")
    centers = problems.site_centers(10.0, 10.0, 16, 2011)
    sub = problems.slab(10.0, 0.2, 2.0, 0.01, stim="face")  # geometry of the sampled sub-slab
    assert sub.n == op.n
    want = sub.sheet.discs_z0(centers, problems.C5_SITE_RADIUS)
    assert np.array_equal(want, nodes)


def test_struct_oracle_equals_csr_oracle():
    import orapy
    for nx, ny, nz in ((6, 5, 4), (2, 2, 3), (3, 7, 1)):
        op = orapy.Slab3DOp(nx, ny, nz, 0.02)
        csr, dt_s = orapy.assemble_slab3d(nx, ny, nz, 0.02, 0.0012, 0.25, op.angles)
        assert dt_s == op.dt_s
        v = np.random.default_rng(nx * 100 + ny).uniform(-90, 40, op.n)
        assert np.array_equal(orapy.diffusion_substep(csr, v, 0.03), op.substep(v, 0.03))


def test_mt19937_64_known_answer_and_product_equality():
    import orapy
    from paper_2011_04747_b200 import problems
    # the C++ standard ([rand.predef]) pins the 10000th output of a default-constructed mt19937_64
    assert int(orapy.mt64_raw(5489, 10000)[-1]) == 9981545732273789042
    assert np.array_equal(orapy.uniform_mt64(2011, 5000, 0.8, 1.2), problems.uniform_mt64(2011, 5000, 0.8, 1.2))


def test_reference_arm_never_imports_the_package():
    """The --impl reference process must not load libcwgpu.so or import paper_2011_04747_b200."""
    code = ("import sys, runpy; sys.argv=['bench.py']; import bench; "
            "bench.host_cpu(); "
            "import orapy; op, nodes, t = bench.oracle_slab('c4'); "
            "assert not any(m.startswith('paper_2011_04747_b200') for m in sys.modules), sorted(sys.modules)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "oracle")]))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    maps = ""  # and no product .so in the process maps of a short reference-arm run
    r = subprocess.run([sys.executable, "-c",
                        "import sys; sys.argv=['bench.py']; import bench, orapy; bench.oracle_slab('c4'); "
                        "print(open('/proc/self/maps').read())"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    maps = r.stdout
    assert "libcwgpu" not in maps


def test_host_cpu_reports_cores():
    import bench
    phys, logical, model = bench.host_cpu()
    assert 1 <= phys <= logical
    assert isinstance(model, str)
