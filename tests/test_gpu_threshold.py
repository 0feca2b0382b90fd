"""diastolic_threshold (stimulus.cpp:115-157) with the probe runs on the GPU,
against the reference's own bisection (oracle/_ref) on the same sheets."""
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # (lx, ly, h, model, strip, window_ms, reference threshold measured with libcwref)
    (1.5, 0.3, 0.05, "aliev-panfilov", 0.1, 200.0, 35.0),
    (1.2, 0.2, 0.04, "ohara2011-epi", 0.08, 40.0, 42.0),
]


@pytest.fixture(scope="module")
def cw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_04747_b200 as cw
    return cw


@pytest.mark.parametrize("case", CASES, ids=["aliev-panfilov", "ohara2011-epi"])
def test_threshold_matches_reference(cw, case):
    lx, ly, h, model, strip, window, expected = case
    sh = cw.Sheet(lx, ly, h, 0.0, d0_myocyte=0.0017, rho=1.0)
    nodes = sh.select("x_le", value=strip)
    thr, probe = cw.diastolic_threshold(sh, cw.make_model(model), nodes, cw.ThresholdOptions(window_ms=window),
                                        return_probe=True)
    import refpy
    if refpy.available():  # the reference itself, same inputs, this host
        r = refpy.Sheet(lx, ly, h, 0.0, d0=0.0017, rho=1.0)
        expected = r.threshold(model, r.select("x_le", value=strip), window_ms=window)
    assert thr == expected
    assert probe == sh.n - 1 or probe == sh.nx1 - 1  # a far corner of the sheet


def test_threshold_errors(cw):
    sh = cw.Sheet(0.5, 0.5, 0.05, 0.0)
    with pytest.raises(cw.ValidationError, match="1 cm"):
        cw.diastolic_threshold(sh, cw.make_model("aliev-panfilov"), sh.select("x_le", value=0.0))
    sh = cw.Sheet(1.5, 0.3, 0.05, 0.0, d0_myocyte=0.0017, rho=1.0)
    with pytest.raises(cw.ValidationError, match="upper bracket"):
        cw.diastolic_threshold(sh, cw.make_model("aliev-panfilov"), sh.select("x_le", value=0.1),
                               cw.ThresholdOptions(window_ms=5.0, upper_factor=8.0))
