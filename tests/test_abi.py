"""The C ABI: libcwgpu.so loads, exports every function include/*.h declares,
and its host-side pieces (rules, slab plan, model metadata) agree with the
oracle. No kernel is launched here (CPU-only container)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for hdr in ("cwgpu.h", "cwgpu_setup.h"):
        txt = open(os.path.join(ROOT, "include", hdr)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names += re.findall(r"\b(cwg_[a-z0-9_]+)\s*\(", txt)
    return sorted(set(names))


def test_all_declared_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 40
    missing = [n for n in decl if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers the same surface
    assert set(decl) == set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


def test_reaction_rules_match_oracle(ora):
    rng = np.random.default_rng(5)
    for _ in range(2000):
        d = float(rng.choice([-1, 1]) * 10 ** rng.uniform(-4, 3))
        sch = cw.Scheme(int(rng.integers(3)))
        k0d = int(rng.integers(1, 4))
        cfg = cw.SchemeConfig(scheme=sch, k0_up=k0d + int(rng.integers(0, 5)), k0_down=k0d)
        km = int(rng.integers(1, 15))
        assert cw.reaction_substeps(d, cfg, km) == ora.reaction_substeps(d, sch.name, cfg.k0_up, cfg.k0_down, km)
        dt, dts = float(rng.uniform(0.005, 0.5)), float(rng.uniform(0.001, 0.3))
        strict = bool(rng.integers(2))
        p = cw.diffusion_substeps(dt, dts, strict, sch)
        assert (p.l, p.dt_ad) == ora.diffusion_substeps(dt, dts, strict, sch.name)


def test_model_metadata(ora):
    for name in cw.registered_model_names() + ["passive"]:
        m = cw.make_model(name)
        assert m.state_count() == ora.state_count(name)
        assert m.stable_step() == ora.stable_step(name)
        assert np.array_equal(m.rest_state(), ora.rest_state(name))
        assert cw.k_max_for(0.1, m) == ora.k_max_for(0.1, name)
    with pytest.raises(cw.ValidationError):
        cw.make_model("hodgkin-huxley")


def test_slab_plan_partitions_rows():
    for ny1 in (2, 7, 101, 201, 1001):
        for world in (1, 2, 3, 4, 8):
            if world > ny1:
                with pytest.raises(cw.ValidationError):
                    cw.slab_plan(ny1, world, 0)
                continue
            spans = [cw.slab_plan(ny1, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == ny1
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_scheme_config_validation():
    with pytest.raises(cw.ValidationError):
        cw.SchemeConfig(dt_ms=0.0).validate()
    with pytest.raises(cw.ValidationError):
        cw.SchemeConfig(k0_up=1, k0_down=2).validate()
    with pytest.raises(cw.ValidationError):
        cw.SchemeConfig(t_end_ms=0.01, dt_ms=0.1).validate()
    assert cw.scheme_from_string("OSTAR") == cw.Scheme.OSTAR
    with pytest.raises(cw.ValidationError):
        cw.scheme_from_string("RK4")


def test_no_cpu_fallback_without_gpu():
    """Without a device the integrator must fail loudly (CWG_ECUDA), never compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    sh = cw.Sheet(0.1, 0.1, 0.05, 0.0)
    setup = cw.SimulationSetup(op=sh.op, models=[cw.make_model("aliev-panfilov")])
    with pytest.raises(cw.DeviceError):
        cw.StrangIntegrator(setup, cw.SchemeConfig(t_end_ms=1.0))
    with pytest.raises(cw.DeviceError):
        cw.diffusion_substep(sh.op, np.zeros(sh.n), 0.01)


def test_protocol_index_validation():
    with pytest.raises(cw.ValidationError):
        cw.ProtocolIndex(cw.Protocol([cw.Stimulus(np.array([0]), 0.0, 0.0, 1.0)]), 4)
    with pytest.raises(cw.ValidationError):
        cw.ProtocolIndex(cw.Protocol([cw.Stimulus(np.array([9]), 0.0, 1.0, 1.0)]), 4)
    with pytest.raises(cw.ValidationError):
        cw.ProtocolIndex(cw.Protocol([cw.Stimulus(np.array([], np.int64), 0.0, 1.0, 1.0)]), 4)
    pi = cw.ProtocolIndex(cw.Protocol([cw.Stimulus(np.array([1, 2]), 0.0, 1.0, 5.0),
                                       cw.Stimulus(np.array([2]), 1.0, 1.0, 7.0, period_ms=3.0)]), 4)
    assert list(pi.node_ptr) == [0, 0, 1, 3, 3]
    assert list(pi.ids) == [0, 0, 1]
    assert math.isnan(pi.period[0]) and pi.period[1] == 3.0
