"""Post-processing metrics (paper_2011_04747_b200/postprocess.py) against the
reference's own postprocess.cpp through libcwref: bit-identical values and the
same validation failures."""
import math

import numpy as np
import pytest

import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import postprocess as pp


def _ap_trace(dt, t0=5.0, shift=0.0, n=None, noise=0.0, seed=0):
    rng = np.random.default_rng(seed)
    t = np.arange(0.0, 400.0, dt) if n is None else np.arange(n) * dt
    up = 1.0 / (1.0 + np.exp(-(t - t0 - shift) / 0.4))
    down = 1.0 / (1.0 + np.exp((t - t0 - shift - 250.0) / 12.0))
    v = -85.0 + 125.0 * up * down + noise * rng.standard_normal(len(t))
    return cw.Trace(0, "p", t, v)


TRACES = [_ap_trace(0.1), _ap_trace(1.0, shift=3.3), _ap_trace(0.25, noise=0.3, seed=4), _ap_trace(0.5, t0=-50.0),
          cw.Trace(0, "flat", np.arange(0, 50.0, 1.0), np.full(50, -80.0)),
          cw.Trace(0, "short", np.array([0.0, 1.0]), np.array([-80.0, 20.0]))]


@pytest.mark.parametrize("k", range(len(TRACES)))
def test_apd90_bitwise(ref, k):
    tr = TRACES[k]
    assert pp.compute_apd90(tr) == ref.compute_apd90(tr.t_ms, tr.v_mv)


@pytest.mark.parametrize("a,b", [(0, 1), (1, 0), (0, 2), (2, 3), (0, 4), (1, 2)])
def test_align_and_diff_bitwise(ref, a, b):
    ta, tb = TRACES[a], TRACES[b]
    try:
        mine = pp.align_and_diff(ta, tb)
    except cw.ValidationError:
        with pytest.raises(ref.RefError):
            ref.align_and_diff(ta.t_ms, ta.v_mv, tb.t_ms, tb.v_mv)
        return
    assert mine == ref.align_and_diff(ta.t_ms, ta.v_mv, tb.t_ms, tb.v_mv)


def test_nrmse_and_cv_bitwise(ref):
    rng = np.random.default_rng(11)
    sheet = cw.Sheet(1.0, 0.5, 0.02, 0.3)
    rs = ref.Sheet(1.0, 0.5, 0.02, 0.3)
    n = sheet.n
    lat = rng.uniform(0, 60, n)
    valid = rng.random(n) > 0.1
    lat2 = lat + rng.normal(0, 0.3, n)
    valid2 = rng.random(n) > 0.2
    m1, m2 = cw.ScalarMap(lat, valid.astype(np.uint8)), cw.ScalarMap(lat2, valid2.astype(np.uint8))
    assert pp.nrmse(m1, m2) == ref.nrmse(lat, valid, lat2, valid2)
    for a, b in [(0, n - 1), (5, 700), (3, 3)]:
        try:
            mine = pp.compute_cv(sheet.coords, m1, a, b)
        except cw.ValidationError:
            with pytest.raises(ref.RefError):
                ref.compute_cv(rs, lat, valid, a, b)
            continue
        if valid[a] and valid[b]:
            assert mine == ref.compute_cv(rs, lat, valid, a, b)
    with pytest.raises(cw.ValidationError):
        pp.nrmse(m1, cw.ScalarMap(lat2, np.zeros(n, np.uint8)))
    with pytest.raises(cw.ValidationError):
        pp.nrmse(cw.ScalarMap(np.full(n, 3.0), np.ones(n, np.uint8)), m2)
