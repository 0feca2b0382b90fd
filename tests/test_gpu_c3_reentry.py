"""BASELINE configs[2] does what it exists for: S1 from the left edge, then the S2 cross-field quadrant
stimulus at 300 ms induces re-entry around the scar (tools/c3_reentry.py, profiles/r02_c3_reentry.txt).
Re-entry = tissue re-activated (an upward 0 mV crossing of a probe trace) after the S2 wave is gone, with no
stimulus on: every S1/S2 activation of the probe grid happens before 320 ms; the re-entrant wave returns to
them at ~550-700 ms and again ~330 ms later."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    return cw


def test_c3_s2_induces_reentry(cw):
    from paper_2011_04747_b200 import problems
    p = problems.c3(t_end=1000.0)
    xs = np.linspace(0.25, 4.75, 7)
    p.probes = [p.sheet.nearest(x, y) for y in xs for x in xs]
    r = cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
    late, s2 = 0, 0
    for tr in r.traces:
        v = tr.v_mv
        t_up = tr.t_ms[np.flatnonzero((v[:-1] < 0.0) & (v[1:] >= 0.0)) + 1]
        s2 += int(np.any((t_up > 300.0) & (t_up < 320.0)))
        late += int(np.sum(t_up > 450.0))
    assert s2 >= 10  # the quadrant fired on S2
    assert late >= 20  # re-entrant activations, no stimulus on
    myo = p.model_of_node == 0
    assert int((r.lat_map.valid & myo).sum()) == int(myo.sum())  # S1 reached every myocyte
