"""Writers of the Python mirror (paper_2011_04747_b200/output.py) produce the
same bytes as the reference's output.cpp / NodeStateArray::save."""
import numpy as np
import pytest

import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import output


@pytest.fixture()
def sheets(ref):
    return cw.Sheet(0.5, 0.3, 0.02, 0.4), ref.Sheet(0.5, 0.3, 0.02, 0.4)


def _same(a, b):
    return open(a, "rb").read() == open(b, "rb").read()


def test_vtk_snapshot_bytes(ref, sheets, tmp_path):
    ours, theirs = sheets
    v = np.random.default_rng(1).uniform(-90, 40, ours.n)
    v[3] = 1e-300
    output.write_vtk_snapshot(ours, v, 12.3456789012, str(tmp_path / "a.vtk"))
    ref.write_vtk_snapshot(theirs, v, 12.3456789012, str(tmp_path / "b.vtk"))
    assert _same(tmp_path / "a.vtk", tmp_path / "b.vtk")


@pytest.mark.parametrize("vtk", [False, True])
def test_map_bytes(ref, sheets, tmp_path, vtk):
    ours, theirs = sheets
    rng = np.random.default_rng(2)
    val = rng.uniform(0, 50, ours.n)
    ok = (rng.random(ours.n) > 0.3).astype(np.uint8)
    m = cw.ScalarMap(val, ok)
    if vtk:
        output.write_map_vtk(ours, m, "LAT", str(tmp_path / "a"))
    else:
        output.write_map_csv(ours, m, str(tmp_path / "a"))
    ref.write_map(theirs, val, ok, "LAT", vtk, str(tmp_path / "b"))
    assert _same(tmp_path / "a", tmp_path / "b")


def test_trace_csv_bytes_and_roundtrip(ref, tmp_path):
    t = np.arange(0, 50.0, 0.1)
    v = np.sin(t) * 80.0 - 10.0
    output.write_trace_csv(cw.Trace(1, "p", t, v), str(tmp_path / "a.csv"))
    ref.write_trace_csv(t, v, str(tmp_path / "b.csv"))
    assert _same(tmp_path / "a.csv", tmp_path / "b.csv")
    back = output.read_trace_csv(str(tmp_path / "a.csv"))
    assert np.array_equal(back.t_ms, t) and np.array_equal(back.v_mv, v)


def test_state_cwstate1_bytes_and_roundtrip(ref, tmp_path):
    models = [cw.make_model("ohara2011-epi"), cw.make_model("maccannell2007")]
    mon = (np.arange(57) % 3 == 0).astype(np.uint8)
    st = cw.make_initial_state(57, models, mon)
    st.v = st.v + np.random.default_rng(3).normal(0, 1, 57)
    output.save_state(st, str(tmp_path / "a.bin"))
    ref.state_save(st.n_nodes, st.stride, st.v, st.s, st.last_dvdt, st.model_of_node, str(tmp_path / "b.bin"))
    assert _same(tmp_path / "a.bin", tmp_path / "b.bin")
    back = output.load_state(str(tmp_path / "a.bin"))
    assert back.n_nodes == 57 and back.stride == st.stride
    assert np.array_equal(back.v, st.v) and np.array_equal(back.s, st.s)
    assert np.array_equal(back.model_of_node, st.model_of_node)
    with pytest.raises(cw.IoError):
        (tmp_path / "bad.bin").write_bytes(b"notastate" * 4)
        output.load_state(str(tmp_path / "bad.bin"))
