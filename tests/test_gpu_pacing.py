"""Batched single-cell pacing on the device (cwg_pace_cells) against the
restated pace_to_steady_state (oracle/cw_oracle.c: cwo_pace, pinned to the
reference in tests/test_golden.py). ionic.cpp:122-165."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_batched_pacing_matches_oracle(ora):
    """Each cell of a cycle-length sweep equals the single-cell oracle run."""
    import paper_2011_04747_b200 as cw
    cls = np.array([250.0, 300.0, 333.3, 400.0, 500.0])
    for model, amp, exact in [("aliev-panfilov", 0.5, True), ("maccannell2007", 10.0, False),
                              ("ohara2011-epi", 80.0, False)]:
        res, errs = cw.pace_cells(model, cls, 2, amp, 1.0)
        dt = cw.make_model(model).stable_step() / 2
        for i, cl in enumerate(cls):
            assert errs[i] is None
            st, mr, apd = ora.pace(model, float(cl), 2, amp, 1.0)
            if exact:
                assert np.array_equal(res[i].state, st) and res[i].max_rel_change == mr
                assert np.array_equal(res[i].apd90_ms, apd, equal_nan=True)
            else:
                np.testing.assert_allclose(res[i].state, st, rtol=1e-8, atol=1e-12)
                assert np.array_equal(np.isnan(res[i].apd90_ms), np.isnan(apd))
                ok = ~np.isnan(apd)
                assert np.all(np.abs(res[i].apd90_ms[ok] - apd[ok]) <= dt * 1.0000001)


def test_pacing_errors_like_reference(ora):
    import paper_2011_04747_b200 as cw
    with pytest.raises(cw.ValidationError, match="n_beats"):
        cw.pace_to_steady_state("ohara2011-epi", 500.0, 0, 80.0, 1.0)
    with pytest.raises(cw.ValidationError, match="cycle length"):
        cw.pace_to_steady_state("ohara2011-epi", -1.0, 2, 80.0, 1.0)
    # a batch with one diverging cell: the others still complete
    res, errs = cw.pace_cells("aliev-panfilov", [500.0, 500.0], 2, [0.5, 1e5], 1.0)
    assert errs[0] is None and isinstance(errs[1], cw.InstabilityError)
    with pytest.raises(ora.OracleInstability) as e:
        ora.pace("aliev-panfilov", 500.0, 2, 1e5, 1.0)
    assert errs[1].time_ms == e.value.t and errs[1].node_index == -1
    assert "|V| > 1000 mV at beat 0" in str(errs[1])


def test_paced_initial_state_runs(ora):
    """A paced state as the initial state of a sheet run (make_initial_state's
    initial_per_model, runner.cpp:78-82)."""
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import problems
    paced = cw.pace_to_steady_state("aliev-panfilov", 500.0, 2, 0.5, 1.0).state
    p = problems.c1(model="aliev-panfilov", t_end=10.0, k0_down=1)
    st = cw.make_initial_state(p.n, [cw.make_model("aliev-panfilov")], p.model_of_node, initial_per_model=[paced])
    assert np.all(st.v == paced[0])
    r = cw.run_simulation(st, p.setup(), p.cfg)
    assert np.all(np.isfinite(r.final_state.v))
