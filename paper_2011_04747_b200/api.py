"""Python mirror of the reference's proj/core interfaces over the cwgpu C ABI.

Names, argument meaning and error behaviour follow cardwave (reference
/root/reference/proj/core/include/cardwave/*.hpp) so that parity tests read
like the reference's own usage:

  reference (C++)                               here
  ---------------------------------------------------------------------------
  Scheme, SchemeConfig          splitting.hpp:19-35   Scheme, SchemeConfig
  reaction_substeps             splitting.hpp:42      reaction_substeps
  DiffusionPlan, diffusion_substeps  :43-51           DiffusionPlan, diffusion_substeps
  k_max_for                     splitting.hpp:54      k_max_for
  StrangIntegrator              splitting.hpp:101-127 StrangIntegrator (GPU)
  run_simulation                splitting.hpp:139     run_simulation (GPU)
  make_initial_state            splitting.hpp:131     make_initial_state
  diffusion_substep             fem.hpp:56            diffusion_substep (GPU)
  CellModel / make_model        ionic.hpp:17-61       CellModel / make_model (rates on GPU)
  NodeStateArray                ionic.hpp:39-55       NodeStateArray
  Stimulus/Protocol/ProtocolIndex stimulus.hpp:17-50  same names
  AssembledOperator             fem.hpp:23-32         AssembledOperator
  build_regular_sheet+assemble  mesh.cpp/fem.cpp      build_sheet (host setup, cwgpu_setup.h)
  ValidationError / InstabilityError errors.hpp       same names

Every compute call runs the sm_100a kernels of libcwgpu.so; there is no CPU
fallback path in this module.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib as L


# ----------------------------------------------------------------------------- errors (errors.hpp)
class ValidationError(RuntimeError):
    """Invalid configuration or arguments (CLI exit code 2)."""


class InstabilityError(RuntimeError):
    """Non-finite state (CLI exit code 3), with the reference's node and time."""

    def __init__(self, msg, node, t_ms):
        super().__init__(msg)
        self.node_index = node
        self.time_ms = t_ms


class IoError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    """CUDA / NCCL failure (no reference equivalent)."""


def _raise(code, err: L.cwg_error):
    msg = err.msg.decode(errors="replace")
    if code == L.CWG_EVALIDATION:
        raise ValidationError(msg)
    if code == L.CWG_EINSTABILITY:
        raise InstabilityError(msg, int(err.node), float(err.t_ms))
    if code == L.CWG_EIO:
        raise IoError(msg)
    raise DeviceError(msg or f"cwgpu error {code}")


def _check(code, err=None):
    if code != L.CWG_OK:
        if err is None:
            err = L.cwg_error(code=code)
            err.msg = L.lib().cwg_last_error()[:255]
        _raise(code, err)


# ----------------------------------------------------------------------------- scheme (splitting.hpp)
class Scheme(enum.IntEnum):
    OST = 0
    OSTAR = 1
    DAETI = 2


def scheme_from_string(name: str) -> Scheme:
    try:
        return Scheme[name]
    except KeyError:
        raise ValidationError(f"unknown scheme '{name}' (expected OST, OSTAR or DAETI)") from None


@dataclass
class SchemeConfig:
    scheme: Scheme = Scheme.DAETI
    dt_ms: float = 0.1
    t_end_ms: float = 500.0
    k0_up: int = 5
    k0_down: int = 1
    strict_substeps: bool = False
    record_interval_ms: float = 1.0
    workers: int = 0  # accepted for interface parity; the GPU path ignores it

    def validate(self):
        if not self.dt_ms > 0.0:
            raise ValidationError("scheme: dt must be positive")
        if not self.t_end_ms >= self.dt_ms:
            raise ValidationError("scheme: T must be >= dt")
        if self.k0_down < 1 or self.k0_up < self.k0_down:
            raise ValidationError("scheme: need k0_up >= k0_down >= 1")
        if not self.record_interval_ms > 0.0:
            raise ValidationError("scheme: record interval must be positive")
        if self.workers < 0:
            raise ValidationError("scheme: workers must be >= 0")


@dataclass
class DiffusionPlan:
    l: int = 1
    dt_ad: float = 0.0


def reaction_substeps(dvdt_prev: float, cfg: SchemeConfig, k_max: int) -> int:
    return L.lib().cwg_reaction_substeps(float(dvdt_prev), int(cfg.scheme), cfg.k0_up, cfg.k0_down, k_max)


def diffusion_substeps(dt_ms: float, dt_s_ms: float, strict: bool, scheme: Scheme) -> DiffusionPlan:
    l, dt_ad = C.c_int(), C.c_double()
    if L.lib().cwg_diffusion_substeps(dt_ms, dt_s_ms, int(strict), int(scheme), C.byref(l), C.byref(dt_ad)):
        raise ValidationError("diffusion sub-steps: dt and dt_s must be positive")
    return DiffusionPlan(l.value, dt_ad.value)


# ----------------------------------------------------------------------------- models (ionic.hpp)
class CellModel:
    """Registry model (make_model, ionic.cpp:59-70); rates() evaluates on the GPU."""

    def __init__(self, name: str, kind: int):
        self._name, self.kind = name, kind

    def name(self):
        return self._name

    def state_count(self):
        return L.lib().cwg_model_state_count(self.kind)

    def stable_step(self):
        return L.lib().cwg_model_stable_step(self.kind)

    def rest_state(self):
        out = np.zeros(self.state_count() + 1)
        L.lib().cwg_model_rest_state(self.kind, L.dp(out))
        return out

    def rates(self, v, s, i_stim, device=0):
        """Batched rates: v[n], s[n, ns], i_stim[n] -> (dv[n], ds[n, ns])."""
        v = np.ascontiguousarray(v, np.float64)
        ns = self.state_count()
        s = np.ascontiguousarray(s, np.float64).reshape(len(v), ns)
        i_stim = np.ascontiguousarray(np.broadcast_to(i_stim, v.shape), np.float64)
        dv = np.zeros_like(v)
        ds = np.zeros_like(s)
        err = L.cwg_error()
        _check(L.lib().cwg_rates(self.kind, len(v), L.dp(v), L.dp(s), L.dp(i_stim), L.dp(dv), L.dp(ds), device,
                                 C.byref(err)), err)
        return dv, ds

    def __repr__(self):
        return f"CellModel({self._name!r})"


def registered_model_names():
    return ["aliev-panfilov", "ohara2011-endo", "ohara2011-epi", "ohara2011-mid", "maccannell2007"]


def make_model(name: str) -> CellModel:
    kind = L.lib().cwg_model_kind_from_name(name.encode())
    if kind < 0:
        raise ValidationError(f"unknown cell model: '{name}'")
    return CellModel(name, kind)


def k_max_for(dt_ms: float, model: CellModel) -> int:
    return L.lib().cwg_k_max_for(dt_ms, model.kind)


@dataclass
class PacingResult:
    """ionic.hpp:63-68: end-diastolic [V, s...] of the final beat, the relative
    change between the last two end-diastolic states, APD90 per beat (NaN: none)."""
    state: np.ndarray
    max_rel_change: float
    apd90_ms: np.ndarray


def pace_cells(model, cycle_lengths_ms, n_beats: int, stim_amplitude, stim_duration_ms, device=0):
    """Batched pace_to_steady_state on the device: one single cell per entry of
    cycle_lengths_ms (amplitude / duration scalars or per-cell arrays), one GPU
    thread each. Returns (results, errors): errors[i] is None or the
    InstabilityError the reference would raise for that cell."""
    m = model if isinstance(model, CellModel) else make_model(model)
    cl = np.ascontiguousarray(np.atleast_1d(np.asarray(cycle_lengths_ms, np.float64)))
    n = len(cl)
    amp = np.ascontiguousarray(np.broadcast_to(np.asarray(stim_amplitude, np.float64), (n,)).copy())
    dur = np.ascontiguousarray(np.broadcast_to(np.asarray(stim_duration_ms, np.float64), (n,)).copy())
    ns = m.state_count()
    st = np.zeros((n, ns + 1))
    apd = np.zeros((n, max(1, int(n_beats))))
    mr = np.zeros(n)
    status = np.zeros(n, np.int32)
    ft = np.zeros(n)
    err = L.cwg_error()
    rc = L.lib().cwg_pace_cells(m.kind, n, L.dp(cl), L.dp(amp), L.dp(dur), int(n_beats), L.dp(st), L.dp(apd),
                                L.dp(mr), status.ctypes.data_as(C.POINTER(C.c_int)), L.dp(ft), device,
                                C.byref(err))
    if rc not in (L.CWG_OK, L.CWG_EINSTABILITY):
        _raise(rc, err)
    results, errors = [], []
    for i in range(n):
        results.append(PacingResult(st[i].copy(), float(mr[i]), apd[i].copy()))
        errors.append(None)
    if rc == L.CWG_EINSTABILITY:
        for i in np.flatnonzero(status != L.CWG_OK):
            # per-cell message as the reference's (ionic.cpp:141-147); the C call reports the first
            errors[i] = InstabilityError(err.msg.decode() if i == np.flatnonzero(status != L.CWG_OK)[0]
                                         else "pacing: diverged", -1, float(ft[i]))
    return results, errors


def pace_to_steady_state(model, cycle_length_ms: float, n_beats: int, stim_amplitude: float,
                         stim_duration_ms: float, device=0) -> PacingResult:
    """pace_to_steady_state (ionic.cpp:122-165) for one cell, on the device."""
    res, errs = pace_cells(model, [cycle_length_ms], n_beats, stim_amplitude, stim_duration_ms, device)
    if errs[0] is not None:
        raise errs[0]
    return res[0]


@dataclass
class NodeStateArray:
    n_nodes: int = 0
    stride: int = 0
    v: np.ndarray = None
    s: np.ndarray = None  # n_nodes * stride, node-major (s[i*stride + k])
    last_dvdt: np.ndarray = None
    model_of_node: np.ndarray = None

    def states_of(self, node):
        return self.s[node * self.stride:(node + 1) * self.stride]

    def copy(self):
        return NodeStateArray(self.n_nodes, self.stride, self.v.copy(), self.s.copy(), self.last_dvdt.copy(),
                              self.model_of_node.copy())


def make_initial_state(n_nodes: int, models: Sequence[CellModel], model_of_node, initial_per_model=None):
    """make_initial_state (splitting.cpp:183-217) with the tag->model map already applied."""
    model_of_node = np.ascontiguousarray(model_of_node, np.uint8)
    if len(model_of_node) != n_nodes:
        raise ValidationError("initial state: model_of_node must cover every node")
    stride = max([1] + [m.state_count() for m in models])
    st = NodeStateArray(n_nodes, stride, np.zeros(n_nodes), np.zeros(n_nodes * stride), np.zeros(n_nodes),
                        model_of_node)
    s2 = st.s.reshape(n_nodes, stride)
    for mid, m in enumerate(models):
        init = None
        if initial_per_model is not None and mid < len(initial_per_model) and initial_per_model[mid] is not None:
            init = np.asarray(initial_per_model[mid], np.float64)
        if init is None:
            init = m.rest_state()
        if len(init) != m.state_count() + 1:
            raise ValidationError(f"initial state: wrong state vector length for model {m.name()}")
        sel = model_of_node == mid
        st.v[sel] = init[0]
        s2[np.ix_(sel, np.arange(m.state_count()))] = init[1:]
    if model_of_node.size and model_of_node.max() >= len(models):
        raise ValidationError("initial state: node has no model")
    return st


# ----------------------------------------------------------------------------- operator + setup
@dataclass
class AssembledOperator:
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    lumped_mass: np.ndarray
    dt_s: float
    grid_nx1: int = 0  # regular-sheet node counts (enables the stencil kernel and y-slabs)
    grid_ny1: int = 0

    def rows(self):
        return len(self.lumped_mass)

    def entry(self, i, j):
        for p in range(self.row_ptr[i], self.row_ptr[i + 1]):
            if self.col[p] == j:
                return self.val[p]
        return 0.0


class DeviceSheetOperator:
    """The operator of a regular sheet assembled ON THE DEVICE (cwg_sheet2d / CWG_OP_SHEET2D):
    build_diffusion_field (fem.cpp:21-51) + assemble (fem.cpp:112-176) + gershgorin_step (fem.cpp:178-192) without
    the host triplet sort or a CSR upload. Acts as SimulationSetup.op. Lumped mass and off-diagonal entries equal
    the reference's bit for bit; a diagonal entry can differ by 1-2 ulp (its four element contributions are summed
    in ascending element order, the reference's in std::sort's tie order). `csr()` returns the assembled CSR."""

    def __init__(self, nx, ny, h, fiber_angle_rad, d0_myocyte, d0_fibrotic, rho, tags=None, elem_scale=None,
                 device=0):
        self._tags = None if tags is None else np.ascontiguousarray(tags, np.int32)
        self._es = None if elem_scale is None else np.ascontiguousarray(elem_scale, np.float64)
        self.desc = L.cwg_sheet2d(nx, ny, h, fiber_angle_rad, d0_myocyte, d0_fibrotic, rho,
                                  None if self._tags is None else self._tags.ctypes.data_as(L._i32p),
                                  None if self._es is None else L.dp(self._es))
        self.grid_nx1, self.grid_ny1 = nx + 1, ny + 1
        self.n = self.grid_nx1 * self.grid_ny1
        self.device = device
        dts = C.c_double()
        err = L.cwg_error()
        _check(L.lib().cwg_sheet2d_assemble(C.byref(self.desc), device, None, None, None, None, C.byref(dts),
                                            C.byref(err)), err)
        self.dt_s = dts.value

    def rows(self):
        return self.n

    def __getattr__(self, name):
        # the CSR views (row_ptr, col, val, lumped_mass, entry) for the entry points that take an
        # AssembledOperator (diffusion_substep, diastolic_threshold, ...): assembled once on demand
        if name in ("row_ptr", "col", "val", "lumped_mass", "entry"):
            if "_csr" not in self.__dict__:
                self.__dict__["_csr"] = self.csr()
            return getattr(self.__dict__["_csr"], name)
        raise AttributeError(name)

    def csr(self) -> AssembledOperator:
        nnz = L.lib().cwg_sheet2d_nnz(C.byref(self.desc))
        rp, col = np.zeros(self.n + 1, np.int64), np.zeros(nnz, np.int64)
        val, mass = np.zeros(nnz), np.zeros(self.n)
        dts = C.c_double()
        err = L.cwg_error()
        _check(L.lib().cwg_sheet2d_assemble(C.byref(self.desc), self.device, L.lp(rp), L.lp(col), L.dp(val),
                                            L.dp(mass), C.byref(dts), C.byref(err)), err)
        return AssembledOperator(rp, col, val, mass, dts.value, self.grid_nx1, self.grid_ny1)


class Sheet:
    """build_regular_sheet (+assign_fibrosis) + build_diffusion_field + assemble.

    assembly="host" (default): the host restatement of the reference's assembly, CSR bit-identical to it.
    assembly="device": only the mesh is built on the host (coordinates, fibrosis tags); the operator is
    assembled on the GPU (DeviceSheetOperator) -- the path for large sheets."""

    def __init__(self, lx_cm, ly_cm, h_cm, fiber_angle_rad=0.0, d0_myocyte=0.0017, d0_fibrotic=0.00066, rho=0.25,
                 fib_fraction=0.0, seed=0, elem_scale=None, assembly="host", device=0):
        lib = L.lib()
        h = C.c_void_p()
        err = L.cwg_error()
        es = None
        if elem_scale is not None:
            self._es = np.ascontiguousarray(elem_scale, np.float64)
            es = L.dp(self._es)
        if assembly == "host":
            rc = lib.cwg_sheet_build(lx_cm, ly_cm, h_cm, fiber_angle_rad, d0_myocyte, d0_fibrotic, rho, fib_fraction,
                                     seed, es, C.byref(h), C.byref(err))
        elif assembly == "device":
            rc = lib.cwg_sheet_mesh(lx_cm, ly_cm, h_cm, fib_fraction, seed, C.byref(h), C.byref(err))
        else:
            raise ValidationError(f"sheet: unknown assembly '{assembly}'")
        _check(rc, err)
        self._h = h
        n = lib.cwg_sheet_nodes(h)
        self.n = n
        self.nx1, self.ny1 = lib.cwg_sheet_nx1(h), lib.cwg_sheet_ny1(h)
        self.n_elements = lib.cwg_sheet_elements(h)
        as_np = np.ctypeslib.as_array
        self.coords = as_np(lib.cwg_sheet_coords(h), (n, 2)).copy()
        self.tags = as_np(lib.cwg_sheet_tags(h), (n,)).copy()
        if assembly == "host":
            nnz = lib.cwg_sheet_nnz(h)
            self.op = AssembledOperator(as_np(lib.cwg_sheet_row_ptr(h), (n + 1,)).copy(),
                                        as_np(lib.cwg_sheet_col(h), (nnz,)).copy(),
                                        as_np(lib.cwg_sheet_val(h), (nnz,)).copy(),
                                        as_np(lib.cwg_sheet_mass(h), (n,)).copy(),
                                        lib.cwg_sheet_dt_s(h), self.nx1, self.ny1)
        else:
            self.op = DeviceSheetOperator(self.nx1 - 1, self.ny1 - 1, h_cm, fiber_angle_rad, d0_myocyte, d0_fibrotic,
                                          rho, self.tags if fib_fraction > 0.0 else None, elem_scale, device)

    def __del__(self):
        if getattr(self, "_h", None) and L._lib is not None:
            L._lib.cwg_sheet_free(self._h)
            self._h = None

    _KINDS = {"x_le": 0, "x_ge": 1, "y_le": 2, "y_ge": 3, "rectangle": 4, "node_set": 5, "disc": 6}

    def select(self, kind, value=0.0, x0=0.0, x1=0.0, y0=0.0, y1=0.0, cx=0.0, cy=0.0, radius=0.0, nodes=()):
        """select_nodes (mesh.cpp:124-180)."""
        prm = np.array([value, x0, x1, y0, y1, cx, cy, radius], np.float64)
        sn = np.array(list(nodes) or [0], np.int64)
        out = np.zeros(self.n, np.int64)
        m = L.lib().cwg_sheet_select(self._h, self._KINDS[kind], L.dp(prm), L.lp(sn), len(nodes), L.lp(out), self.n)
        if m < 0:
            raise ValidationError("selector: invalid selection")
        return out[:m].copy()

    def nearest(self, x, y):
        return L.lib().cwg_sheet_nearest(self._h, x, y)


def build_sheet(*args, **kw) -> Sheet:
    return Sheet(*args, **kw)


def _cells(length, h, axis):
    q = length / h
    r = round(q)
    if r < 1 or abs(q - r) > 1e-9 * max(1.0, q):
        raise ValidationError(f"mesh: {axis} extent {length} cm is not a positive multiple of h = {h} cm")
    return int(r)


class Slab3D:
    """3D slab (EXTENSION for BASELINE configs 4-5; the reference is 2D only).

    (nx+1) x (ny+1) x (nz+1) nodes at spacing h, node index
    (iy*(nz+1) + iz)*(nx+1) + ix (y outermost: y-slabs are contiguous),
    trilinear hexahedra with 2x2x2 Gauss and row-sum lumped mass, transmural
    fibre rotation linear in z from angle_endo (z = 0) to angle_epi (z = lz)
    evaluated at each element layer's mid-plane, D_t = rho * D_l. The device
    keeps 27 coefficients per node class (cwgpu_setup.h) instead of a CSR.
    Acts as the operator object of SimulationSetup.op.
    """

    def __init__(self, lx, ly, lz, h, d_long=0.0012, rho=0.25, angle_endo_deg=60.0, angle_epi_deg=-60.0):
        self.nx, self.ny, self.nz = _cells(lx, h, "x"), _cells(ly, h, "y"), _cells(lz, h, "z")
        self.h, self.d_long, self.rho = h, d_long, rho
        self.nx1, self.ny1, self.nz1 = self.nx + 1, self.ny + 1, self.nz + 1
        self.n = self.nx1 * self.ny1 * self.nz1
        self.plane = self.nx1 * self.nz1
        self.angles = np.deg2rad(angle_endo_deg + (angle_epi_deg - angle_endo_deg) * (np.arange(self.nz) + 0.5) / self.nz)
        self.s3d = L.cwg_struct3d(self.nx, self.ny, self.nz, h, d_long, rho, L.dp(self.angles))
        ncls = 9 * self.nz1
        self.coef = np.zeros(ncls * 27)
        self.mass = np.zeros(ncls)
        self.dt_s = L.lib().cwg_struct3d_tables(C.byref(self.s3d), L.dp(self.coef), L.dp(self.mass))
        if not self.dt_s > 0:
            raise ValidationError("slab: invalid parameters")
        self.op = self

    def rows(self):
        return self.n

    def index(self, ix, iy, iz):
        return (np.asarray(iy) * self.nz1 + np.asarray(iz)) * self.nx1 + np.asarray(ix)

    def face_z0(self):
        """Endocardial face (z = 0) node indices, ascending."""
        iy, ix = np.meshgrid(np.arange(self.ny1), np.arange(self.nx1), indexing="ij")
        return np.sort(self.index(ix, iy, 0).ravel())

    def discs_z0(self, centers, radius):
        """z = 0 nodes within `radius` of any (cx, cy) (1e-9 cm inclusive, like select_nodes)."""
        iy, ix = np.meshgrid(np.arange(self.ny1), np.arange(self.nx1), indexing="ij")
        x, y = ix * self.h, iy * self.h
        sel = np.zeros(ix.shape, bool)
        for cx, cy in centers:
            sel |= np.sqrt((x - cx) ** 2 + (y - cy) ** 2) <= radius + 1e-9
        return np.sort(self.index(ix[sel], iy[sel], 0))

    def nearest(self, x, y, z):
        ix = min(max(int(round(x / self.h)), 0), self.nx)
        iy = min(max(int(round(y / self.h)), 0), self.ny)
        iz = min(max(int(round(z / self.h)), 0), self.nz)
        return int(self.index(ix, iy, iz))


# ----------------------------------------------------------------------------- stimulus (stimulus.hpp)
@dataclass
class Stimulus:
    nodes: np.ndarray
    t_start_ms: float = 0.0
    duration_ms: float = 1.0
    amplitude: float = 0.0
    period_ms: Optional[float] = None
    label: str = ""

    def active_at(self, t_ms):
        if t_ms < self.t_start_ms:
            return False
        if self.period_ms is None:
            return t_ms < self.t_start_ms + self.duration_ms
        return math.fmod(t_ms - self.t_start_ms, self.period_ms) < self.duration_ms


@dataclass
class Protocol:
    entries: List[Stimulus] = field(default_factory=list)


class ProtocolIndex:
    """Compiled per-node view (stimulus.cpp:17-31), flattened for the device."""

    def __init__(self, protocol: Protocol, n_nodes: int):
        es = protocol.entries
        for st in es:
            if not st.duration_ms > 0.0:
                raise ValidationError("stimulus: duration must be positive")
            if not math.isfinite(st.amplitude):
                raise ValidationError("stimulus: amplitude must be finite")
            if len(st.nodes) == 0:
                raise ValidationError("stimulus: node set is empty")
            nd = np.asarray(st.nodes, np.int64)
            if nd.min() < 0 or nd.max() >= n_nodes:
                bad = nd[(nd < 0) | (nd >= n_nodes)][0]
                raise ValidationError(f"stimulus: node {bad} out of range")
        self.n_entries = len(es)
        # per-node entry lists in protocol order (stimulus.cpp:17-31), vectorised
        if es:
            nodes = np.concatenate([np.asarray(st.nodes, np.int64) for st in es])
            eids = np.concatenate([np.full(len(st.nodes), e, np.int32) for e, st in enumerate(es)])
            order = np.lexsort((eids, nodes))
            counts = np.bincount(nodes, minlength=n_nodes)
            self.ids = np.ascontiguousarray(eids[order])
        else:
            counts = np.zeros(n_nodes, np.int64)
            self.ids = np.zeros(1, np.int32)
        self.node_ptr = np.zeros(n_nodes + 1, np.int32)
        np.cumsum(counts, out=self.node_ptr[1:])
        self.t_start = np.array([s.t_start_ms for s in es] or [0.0])
        self.duration = np.array([s.duration_ms for s in es] or [1.0])
        self.amplitude = np.array([s.amplitude for s in es] or [0.0])
        self.period = np.array([math.nan if s.period_ms is None else s.period_ms for s in es] or [math.nan])

    def empty(self):
        return self.n_entries == 0


@dataclass
class Probe:
    node: int = -1
    name: str = ""


@dataclass
class Trace:
    node: int
    name: str
    t_ms: np.ndarray
    v_mv: np.ndarray


@dataclass
class ScalarMap:
    value: np.ndarray
    valid: np.ndarray


@dataclass
class TimingBreakdown:
    total_ms: float = 0.0
    reaction_ms: float = 0.0
    diffusion_ms: float = 0.0
    recording_ms: float = 0.0


@dataclass
class SimulationSetup:
    op: AssembledOperator = None
    models: List[CellModel] = field(default_factory=list)
    protocol: Optional[ProtocolIndex] = None
    probes: List[Probe] = field(default_factory=list)
    lat_threshold_mv: float = 0.0
    map_interval_ms: float = 1.0
    gkr_scale: Optional[np.ndarray] = None  # extension: per-node ORd GKr multiplier
    # splitting.hpp:90-93: snapshot cadence + callbacks
    snapshot_interval_ms: float = 0.0       # 0: no snapshots
    on_snapshot: Optional[Callable[[float, np.ndarray], None]] = None
    progress_every: int = 0
    on_progress: Optional[Callable[[int, float, "TimingBreakdown"], None]] = None


@dataclass
class SimulationResult:
    traces: List[Trace]
    lat_map: ScalarMap
    apd90_map: ScalarMap
    timing: TimingBreakdown
    k_histogram: np.ndarray
    dt_effective: float
    dt_s: float
    plan: DiffusionPlan
    n_steps: int
    final_state: NodeStateArray


# ----------------------------------------------------------------------------- the GPU integrator
class StrangIntegrator:
    """StrangIntegrator (splitting.hpp:101-127) on one B200 (or one y-slab of N).

    The node state lives on the device; advance() mirrors the reference's
    in-place mutation of the caller's NodeStateArray (upload when the state
    object changed, download after the step).
    """

    def __init__(self, setup: SimulationSetup, cfg: SchemeConfig, model_of_node=None, device=0, rank=0, world=1,
                 nccl_id: bytes = None, op_kind=L.OP_AUTO):
        cfg.validate()
        if setup.op is None:
            raise ValidationError("integrator: missing assembled operator")
        if not setup.models:
            raise ValidationError("integrator: no cell models")
        self.setup, self.cfg = setup, cfg
        op = setup.op
        n = op.rows()
        if model_of_node is None:
            model_of_node = np.zeros(n, np.uint8)
        keep = {}
        p = L.cwg_problem()
        p.n = n
        p.dt_s = op.dt_s
        if isinstance(op, Slab3D):
            keep["s3d"] = op.s3d
            p.op_kind = L.OP_STRUCT3D
            p.s3d = C.pointer(op.s3d)
        elif isinstance(op, DeviceSheetOperator):
            keep["sheet2d"] = op
            p.op_kind = L.OP_SHEET2D
            p.sheet2d = C.pointer(op.desc)
        else:
            keep["rp"] = np.ascontiguousarray(op.row_ptr, np.int64)
            keep["col"] = np.ascontiguousarray(op.col, np.int64)
            keep["val"] = np.ascontiguousarray(op.val, np.float64)
            keep["mass"] = np.ascontiguousarray(op.lumped_mass, np.float64)
            p.row_ptr, p.col, p.val, p.lumped_mass = L.lp(keep["rp"]), L.lp(keep["col"]), L.dp(keep["val"]), L.dp(
                keep["mass"])
            p.op_kind = op_kind
            p.grid_nx1, p.grid_ny1 = op.grid_nx1, op.grid_ny1
        keep["kinds"] = np.array([m.kind for m in setup.models], np.int32)
        p.n_models = len(setup.models)
        p.model_kind = keep["kinds"].ctypes.data_as(L._ip)
        keep["mon"] = np.ascontiguousarray(model_of_node, np.uint8)
        p.model_of_node = keep["mon"].ctypes.data_as(L._u8p)
        if setup.gkr_scale is not None:
            keep["gkr"] = np.ascontiguousarray(setup.gkr_scale, np.float64)
            p.gkr_scale = L.dp(keep["gkr"])
        pi = setup.protocol
        if pi is not None and not pi.empty():
            for k in ("node_ptr", "ids", "t_start", "duration", "amplitude", "period"):
                keep["st_" + k] = getattr(pi, k)
            p.n_stim = pi.n_entries
            p.stim_t_start, p.stim_duration = L.dp(pi.t_start), L.dp(pi.duration)
            p.stim_amplitude, p.stim_period = L.dp(pi.amplitude), L.dp(pi.period)
            p.stim_node_ptr = pi.node_ptr.ctypes.data_as(L._i32p)
            p.stim_ids = pi.ids.ctypes.data_as(L._i32p)
        keep["probes"] = np.array([pr.node for pr in setup.probes] or [0], np.int64)
        p.n_probes = len(setup.probes)
        p.probes = L.lp(keep["probes"])
        p.lat_threshold_mv = setup.lat_threshold_mv
        p.map_interval_ms = setup.map_interval_ms
        p.scheme, p.dt_ms, p.t_end_ms = int(cfg.scheme), cfg.dt_ms, cfg.t_end_ms
        p.k0_up, p.k0_down, p.strict_substeps = cfg.k0_up, cfg.k0_down, int(cfg.strict_substeps)
        p.record_interval_ms = cfg.record_interval_ms
        p.device, p.rank, p.world = device, rank, world
        if world > 1 and nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValidationError("placement: world > 1 needs a 128-byte NCCL unique id")
            keep["nid"] = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            p.nccl_id = C.cast(keep["nid"], C.POINTER(C.c_ubyte))
        # (world > 1 without an id: only the CWG_LOOPBACK testing mode, cwg_loopback_steps)
        err = L.cwg_error()
        h = C.c_void_p()
        _check(L.lib().cwg_create(C.byref(p), C.byref(h), C.byref(err)), err)
        self._h = h
        self._keep = keep
        self.n = n
        self.rank, self.world = rank, world
        info = L.cwg_info()
        L.lib().cwg_get_info(h, C.byref(info))
        self.info = info
        self._state_id = None

    def close(self):
        if getattr(self, "_h", None) and L._lib is not None:
            L._lib.cwg_destroy(self._h)
            self._h = None

    __del__ = close

    def set_scheme(self, cfg: SchemeConfig):
        """Reconfigure scheme / dt / T / k0 on the same device-resident operator
        (cwg_set_scheme; cli_compare, runner.cpp:254-324). The record interval
        given at construction is kept. Upload a state and run_begin() next."""
        cfg.validate()
        err = L.cwg_error()
        _check(L.lib().cwg_set_scheme(self._h, int(cfg.scheme), cfg.dt_ms, cfg.t_end_ms, cfg.k0_up, cfg.k0_down,
                                      int(cfg.strict_substeps), C.byref(err)), err)
        self.cfg = cfg
        info = L.cwg_info()
        L.lib().cwg_get_info(self._h, C.byref(info))
        self.info = info
        self._state_id = None

    # --- reference accessors
    def dt_effective(self):
        return self.info.dt_effective

    def plan(self):
        return DiffusionPlan(self.info.l, self.info.dt_ad)

    def k_max_global(self):
        return self.info.k_max_global

    def k_histogram(self):
        h = np.zeros(self.info.k_max_global + 1, np.int64)
        _check(L.lib().cwg_get_khist(self._h, L.lp(h), len(h)))
        return h

    def timing(self):
        r, d, rec = C.c_double(), C.c_double(), C.c_double()
        L.lib().cwg_get_timing(self._h, C.byref(r), C.byref(d), C.byref(rec))
        return TimingBreakdown(r.value + d.value + rec.value, r.value, d.value, rec.value)

    def launch_count(self):
        return L.lib().cwg_launch_count(self._h)

    def stream(self):
        return L.lib().cwg_stream(self._h)

    def set_stream(self, cuda_stream_handle):
        _check(L.lib().cwg_set_stream(self._h, cuda_stream_handle))

    # --- state movement
    def init_rest(self):
        """make_initial_state from rest states directly on the device (no host arrays)."""
        _check(L.lib().cwg_init_rest_state(self._h))
        self._state_id = None

    def upload(self, state: NodeStateArray):
        _check(L.lib().cwg_upload_state(self._h, L.dp(state.v), L.dp(state.s), state.stride, L.dp(state.last_dvdt)))
        self._state_id = id(state)

    def download(self, state: NodeStateArray):
        _check(L.lib().cwg_download_state(self._h, L.dp(state.v), L.dp(state.s), state.stride, L.dp(state.last_dvdt)))

    def advance(self, state: NodeStateArray, t_ms: float, step_index: int, n_steps: int, sync_state=True):
        """One outer step; mutates `state` in place like splitting.cpp:171-181."""
        if self._state_id != id(state):
            self.upload(state)
        err = L.cwg_error()
        rc = L.lib().cwg_advance(self._h, t_ms, step_index, n_steps, C.byref(err))
        if sync_state or rc == L.CWG_EINSTABILITY:
            self.download(state)
        _check(rc, err)

    # --- run_simulation pieces
    def run_begin(self):
        _check(L.lib().cwg_run_begin(self._h))

    def run_steps(self, first, count):
        _check(L.lib().cwg_run_steps(self._h, first, count))

    def run_sync(self):
        err = L.cwg_error()
        _check(L.lib().cwg_run_sync(self._h, C.byref(err)), err)

    def traces(self):
        ns, npb = self.info.n_samples, len(self.setup.probes)
        t = np.zeros(ns)
        v = np.zeros(max(npb, 1) * ns)
        _check(L.lib().cwg_get_traces(self._h, L.dp(t), L.dp(v)))
        return t, v[: npb * ns].reshape(npb, ns)

    @staticmethod
    def _map_buffers(n, out):
        """(lat, apd) ScalarMaps to fill: `out` (e.g. pinned host arrays reused across runs; value float64[n],
        valid bool[n], written in place) or fresh arrays."""
        if out is None:
            out = (ScalarMap(np.empty(n), np.empty(n, bool)), ScalarMap(np.empty(n), np.empty(n, bool)))
        for m in out:
            if (m.value.dtype != np.float64 or m.valid.dtype != np.bool_ or m.value.shape != (n,)
                    or m.valid.shape != (n,) or not m.value.flags.c_contiguous or not m.valid.flags.c_contiguous):
                raise ValidationError("maps: output arrays must be contiguous float64[n] / bool[n]")
        return out

    def gather(self, state: NodeStateArray, maps_out=None):
        """The global final state and LAT/APD maps on every rank (cwg_gather_result; collective for world > 1):
        returns (lat_map, apd90_map) and fills `state` (global arrays)."""
        lat, apd = self._map_buffers(self.n, maps_out)
        _check(L.lib().cwg_gather_result(self._h, L.dp(state.v), L.dp(state.s), state.stride, L.dp(state.last_dvdt),
                                         L.dp(lat.value), lat.valid.ctypes.data_as(L._u8p), L.dp(apd.value),
                                         apd.valid.ctypes.data_as(L._u8p)))
        return lat, apd

    def maps(self, out=None):
        """LAT / APD90 maps of the owned nodes (NaN where a map has no value); `out`: see _map_buffers."""
        lat, apd = self._map_buffers(self.info.n_local, out)
        _check(L.lib().cwg_get_maps(self._h, L.dp(lat.value), lat.valid.ctypes.data_as(L._u8p), L.dp(apd.value),
                                    apd.valid.ctypes.data_as(L._u8p)))
        return lat, apd


def round_half_away(x: float) -> int:
    """std::llround."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def _run_with_callbacks(integ, state, setup, n_steps, dt, every_snap, every_prog, t0):
    """The run loop with on_snapshot / on_progress (splitting.cpp:265-283).
    Snapshots are asynchronous (cwg_snapshot_begin): snapshot N's copy drains
    and its callback runs while the device computes the next chunk; a failure
    before the snapshot point raises instead of delivering it."""
    import time
    lib = L.lib()
    snap = None
    if every_snap:
        snap = np.zeros(state.n_nodes)
        registered = lib.cwg_host_register(snap.ctypes.data, snap.nbytes) == L.CWG_OK
        setup.on_snapshot(0.0, state.v.copy())
    pending, pending_t = False, 0.0

    def deliver():
        err = L.cwg_error()
        _check(lib.cwg_snapshot_wait(integ._h, C.byref(err)), err)
        setup.on_snapshot(pending_t, snap.copy())

    try:
        s = 0
        while s < n_steps:
            nxt = n_steps
            if every_snap:
                nxt = min(nxt, (s // every_snap + 1) * every_snap)
            if every_prog:
                nxt = min(nxt, (s // every_prog + 1) * every_prog)
            integ.run_steps(s, nxt - s)
            if pending:
                pending = False
                deliver()
            s = nxt
            if every_snap and s % every_snap == 0:
                _check(lib.cwg_snapshot_begin(integ._h, L.dp(snap)))
                pending, pending_t = True, s * dt
            if (every_prog and s % every_prog == 0) or s == n_steps:
                if pending:
                    pending = False
                    deliver()
                integ.run_sync()
                if every_prog and s % every_prog == 0:
                    tb = integ.timing()
                    tb.total_ms = (time.perf_counter() - t0) * 1e3
                    setup.on_progress(s, s * dt, tb)
        if pending:
            pending = False
            deliver()
    finally:
        if pending:  # an exception left a copy in flight: drain it before the buffer goes away
            lib.cwg_snapshot_wait(integ._h, None)
        if every_snap and registered:
            lib.cwg_host_unregister(snap.ctypes.data)


def run_simulation(state: NodeStateArray, setup: SimulationSetup, cfg: SchemeConfig, device=0,
                   integrator: StrangIntegrator = None, final_state_out: NodeStateArray = None,
                   maps_out=None) -> SimulationResult:
    """run_simulation (splitting.cpp:219-294) on the GPU; raises InstabilityError like the reference.

    The reference takes `state` by value and moves it into result.final_state; here the caller's arrays
    are left untouched and the final state is downloaded into fresh arrays -- or into `final_state_out`
    (e.g. pinned host buffers a caller reuses across runs), which is then returned as final_state; likewise
    `maps_out` = (lat_map, apd90_map) ScalarMaps receive the LAT / APD90 maps."""
    import time
    t0 = time.perf_counter()
    integ = integrator or StrangIntegrator(setup, cfg, model_of_node=state.model_of_node, device=device)
    integ.upload(state)
    integ.run_begin()
    n_steps, dt = integ.info.n_steps, integ.dt_effective()
    every_snap = (max(1, int(round_half_away(setup.snapshot_interval_ms / dt)))
                  if setup.snapshot_interval_ms > 0.0 and setup.on_snapshot else 0)
    every_prog = setup.progress_every if setup.progress_every > 0 and setup.on_progress else 0
    if not every_snap and not every_prog:
        integ.run_steps(0, n_steps)
        integ.run_sync()
    else:
        _run_with_callbacks(integ, state, setup, n_steps, dt, every_snap, every_prog, t0)
    if final_state_out is not None:
        final = final_state_out
    else:  # every element is overwritten (all ranks' slabs gathered for world > 1): no copy of the input
        final = NodeStateArray(state.n_nodes, state.stride, np.empty_like(state.v), np.empty_like(state.s),
                               np.empty_like(state.last_dvdt), state.model_of_node.copy())
    t, v = integ.traces()
    if integ.world > 1:  # one global SimulationResult on every rank (splitting.cpp:286-293)
        lat, apd = integ.gather(final, maps_out)
    else:
        integ.download(final)
        lat, apd = integ.maps(maps_out)
    traces = [Trace(pr.node, pr.name, t.copy(), v[q].copy()) for q, pr in enumerate(setup.probes)]
    tb = TimingBreakdown(total_ms=(time.perf_counter() - t0) * 1e3)
    return SimulationResult(traces, lat, apd, tb, integ.k_histogram(), integ.dt_effective(), setup.op.dt_s,
                            integ.plan(), integ.info.n_steps, final)


def diffusion_substep(op: AssembledOperator, v, dt_sub: float, device=0):
    """diffusion_substep (fem.cpp:194-207) on the GPU, bit-identical to the reference."""
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty_like(v)
    rp = np.ascontiguousarray(op.row_ptr, np.int64)
    col = np.ascontiguousarray(op.col, np.int64)
    val = np.ascontiguousarray(op.val, np.float64)
    mass = np.ascontiguousarray(op.lumped_mass, np.float64)
    err = L.cwg_error()
    _check(L.lib().cwg_diffusion_substep(len(mass), L.lp(rp), L.lp(col), L.dp(val), L.dp(mass), L.dp(v), dt_sub,
                                         L.dp(out), device, C.byref(err)), err)
    return out


def slab_plan(ny1: int, world: int, rank: int):
    b, e = C.c_int64(), C.c_int64()
    if L.lib().cwg_slab_plan(ny1, world, rank, C.byref(b), C.byref(e)):
        raise ValidationError("placement: fewer rows than ranks")
    return b.value, e.value


@dataclass
class ThresholdOptions:
    """stimulus.hpp:60-67"""
    duration_ms: float = 1.0
    upper_factor: float = 1000.0
    initial_guess: float = 1.0
    rel_tol: float = 0.05
    window_ms: float = 50.0
    dt_ms: float = 0.05


def diastolic_threshold(sheet: Sheet, model: CellModel, stim_nodes, options: ThresholdOptions = None, device=0,
                        return_probe=False):
    """diastolic_threshold (stimulus.cpp:115-157) with every probe run on the GPU."""
    o = options or ThresholdOptions()
    op = sheet.op
    p = L.cwg_problem()
    keep = [np.ascontiguousarray(op.row_ptr, np.int64), np.ascontiguousarray(op.col, np.int64),
            np.ascontiguousarray(op.val, np.float64), np.ascontiguousarray(op.lumped_mass, np.float64)]
    p.n = op.rows()
    p.row_ptr, p.col, p.val, p.lumped_mass = L.lp(keep[0]), L.lp(keep[1]), L.dp(keep[2]), L.dp(keep[3])
    p.dt_s = op.dt_s
    p.op_kind = L.OP_AUTO
    p.grid_nx1, p.grid_ny1 = op.grid_nx1, op.grid_ny1
    kinds = np.array([model.kind], np.int32)
    mon = np.zeros(p.n, np.uint8)
    p.n_models, p.model_kind, p.model_of_node = 1, kinds.ctypes.data_as(L._ip), mon.ctypes.data_as(L._u8p)
    p.scheme, p.dt_ms, p.t_end_ms, p.k0_up, p.k0_down, p.record_interval_ms = 0, 0.1, 0.1, 1, 1, 1.0
    p.device, p.world = device, 1
    xy = np.ascontiguousarray(sheet.coords, np.float64)
    sn = np.ascontiguousarray(stim_nodes, np.int64)
    opt = L.cwg_threshold_options(o.duration_ms, o.upper_factor, o.initial_guess, o.rel_tol, o.window_ms, o.dt_ms)
    thr, probe, err = C.c_double(), C.c_int64(-1), L.cwg_error()
    _check(L.lib().cwg_diastolic_threshold(C.byref(p), L.dp(xy), L.lp(sn), len(sn), C.byref(opt), C.byref(thr),
                                            C.byref(probe), C.byref(err)), err)
    return (thr.value, probe.value) if return_probe else thr.value
