"""Result writers of the Python mirror, byte-compatible with the reference's
output.cpp / ionic.cpp (host-side I/O of data the device path produced):

* write_vtk_snapshot   (output.cpp:31-55)  legacy ASCII VTK, quads, V per point
* write_map_csv        (output.cpp:57-67)  node,x_cm,y_cm,value_ms,valid
* write_map_vtk        (output.cpp:69-90)  invalid nodes as nan
* write_trace_csv / read_trace_csv (output.cpp:92-115)
* save_state / load_state: NodeStateArray in the "cwstate1" binary format
  (ionic.cpp:13-57)

Snapshots come from run_simulation's on_snapshot callback, which the device
path feeds asynchronously (cwg_snapshot_begin) so writing overlaps the run.
"""
import numpy as np

from .api import IoError, NodeStateArray, ScalarMap, Trace, ValidationError


def _quads(sheet):
    nx, ny, w = sheet.nx1 - 1, sheet.ny1 - 1, sheet.nx1
    iy, ix = np.meshgrid(np.arange(ny, dtype=np.int64), np.arange(nx, dtype=np.int64), indexing="ij")
    n0 = (iy * w + ix).ravel()
    return np.stack([n0, n0 + 1, n0 + 1 + w, n0 + w], axis=1)  # build_regular_sheet element order (mesh.cpp:90)


def _g9(x):
    return "%.9g" % x


def _grid_header(f, sheet):
    n = sheet.n
    f.write("POINTS %d double\n" % n)
    f.write("".join("%s %s 0\n" % (_g9(x), _g9(y)) for x, y in sheet.coords))
    q = _quads(sheet)
    ne = len(q)
    f.write("CELLS %d %d\n" % (ne, 5 * ne))
    f.write("".join("4 %d %d %d %d\n" % tuple(e) for e in q))
    f.write("CELL_TYPES %d\n" % ne)
    f.write("9\n" * ne)
    f.write("POINT_DATA %d\n" % n)


def _open(path):
    try:
        return open(path, "w", newline="\n")
    except OSError as e:
        raise IoError("cannot open for write: " + path) from e


def write_vtk_snapshot(sheet, v, t_ms: float, path: str):
    if len(v) != sheet.n:
        raise ValidationError("vtk: field length does not match node count")
    with _open(path) as f:
        f.write("# vtk DataFile Version 3.0\n")
        f.write("transmembrane potential at t = %s ms\n" % _g9(t_ms))
        f.write("ASCII\nDATASET UNSTRUCTURED_GRID\n")
        _grid_header(f, sheet)
        f.write("SCALARS V double 1\nLOOKUP_TABLE default\n")
        f.write("".join(_g9(x) + "\n" for x in np.asarray(v, np.float64)))


def write_map_csv(sheet, m: ScalarMap, path: str):
    if len(m.value) != sheet.n:
        raise ValidationError("map csv: size does not match node count")
    with _open(path) as f:
        f.write("node,x_cm,y_cm,value_ms,valid\n")
        f.write("".join("%d,%.17g,%.17g,%.17g,%d\n" % (i, xy[0], xy[1], val if ok else 0.0, 1 if ok else 0)
                        for i, (xy, val, ok) in enumerate(zip(sheet.coords, m.value, m.valid))))


def write_map_vtk(sheet, m: ScalarMap, name: str, path: str):
    if len(m.value) != sheet.n:
        raise ValidationError("map vtk: size does not match node count")
    with _open(path) as f:
        f.write("# vtk DataFile Version 3.0\n%s map\nASCII\nDATASET UNSTRUCTURED_GRID\n" % name)
        _grid_header(f, sheet)
        f.write("SCALARS %s double 1\nLOOKUP_TABLE default\n" % name)
        f.write("".join((_g9(val) if ok else "nan") + "\n" for val, ok in zip(m.value, m.valid)))


def write_trace_csv(trace: Trace, path: str):
    with _open(path) as f:
        f.write("t_ms,v_mv\n")
        f.write("".join("%.17g,%.17g\n" % (t, v) for t, v in zip(trace.t_ms, trace.v_mv)))


def read_trace_csv(path: str) -> Trace:
    try:
        lines = open(path).read().splitlines()
    except OSError as e:
        raise IoError("trace csv: cannot open " + path) from e
    t, v = [], []
    for line in lines[1:]:
        if "," not in line:
            continue
        a, b = line.split(",", 1)
        t.append(float(a))
        v.append(float(b))
    return Trace(-1, "", np.array(t), np.array(v))


_MAGIC = b"cwstate1"


def save_state(state: NodeStateArray, path: str):
    """NodeStateArray::save: magic, n_nodes, stride (int64), v, s, last_dvdt, model_of_node."""
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(np.array([state.n_nodes, state.stride], np.int64).tobytes())
            f.write(np.ascontiguousarray(state.v, np.float64).tobytes())
            f.write(np.ascontiguousarray(state.s, np.float64).tobytes())
            f.write(np.ascontiguousarray(state.last_dvdt, np.float64).tobytes())
            f.write(np.ascontiguousarray(state.model_of_node, np.uint8).tobytes())
    except OSError as e:
        raise IoError("state: cannot open for write: " + path) from e


def load_state(path: str) -> NodeStateArray:
    try:
        b = open(path, "rb").read()
    except OSError as e:
        raise IoError("state: cannot open for read: " + path) from e
    if b[:8] != _MAGIC:
        raise IoError("state: bad magic in " + path)
    n, stride = (int(x) for x in np.frombuffer(b[8:24], np.int64))
    need = 24 + 8 * (n + n * stride + n) + n
    if len(b) < need:
        raise IoError("state: truncated file: " + path)
    o = 24
    v = np.frombuffer(b, np.float64, n, o).copy()
    o += 8 * n
    s = np.frombuffer(b, np.float64, n * stride, o).copy()
    o += 8 * n * stride
    last = np.frombuffer(b, np.float64, n, o).copy()
    o += 8 * n
    mon = np.frombuffer(b, np.uint8, n, o).copy()
    st = NodeStateArray(n, stride, v, s, last, mon)
    return st
