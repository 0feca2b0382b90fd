"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the C restatement oracle.

oracle/cw_oracle.c restates the reference hot path (cardwave splitting.cpp,
fem.cpp:194-207, stimulus.cpp:33-45, the cell models, postprocess.cpp:18-66).
This module adds `run_simulation`, a restatement of the reference driver loop
(splitting.cpp:171-294) over those C kernels. It is the checker for the CUDA
path in tests/ and in __graft_entry__.smoke(); the product never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcworacle.so")

MODEL_KINDS = {"aliev-panfilov": 0, "ohara2011-endo": 1, "ohara2011-epi": 2, "ohara2011-mid": 3,
               "maccannell2007": 4, "passive": 5}
SCHEMES = {"OST": 0, "OSTAR": 1, "DAETI": 2}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        D, I64, I = C.c_double, C.c_int64, C.c_int
        dp, lp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int)
        u8p = C.POINTER(C.c_uint8)
        sig = {
            "cwo_state_count": (I, [I]),
            "cwo_stable_step": (D, [I]),
            "cwo_rest_state": (None, [I, dp]),
            "cwo_rates": (None, [I, D, dp, D, D, dp, dp]),
            "cwo_rates_batch": (None, [I, I64, dp, dp, dp, dp, dp]),
            "cwo_pace": (I, [I, C.c_double, I, C.c_double, C.c_double, dp, dp, dp, C.POINTER(C.c_int), dp]),
            "cwo_reaction_substeps": (I, [D, I, I, I, I]),
            "cwo_diffusion_substeps": (I, [D, D, I, I, ip, dp]),
            "cwo_k_max_for": (I, [D, D]),
            "cwo_stim_current": (D, [C.c_void_p, I64, D]),
            "cwo_diffusion_substep_csr": (None, [I64, lp, lp, dp, dp, dp, D, dp]),
            "cwo_reaction_step": (I64, [I64, I, dp, dp, dp, u8p, ip, ip, dp, C.c_void_p, I, I, I, D, D, lp, dp]),
            "cwo_detector_init": (None, [C.c_void_p, I64, D]),
            "cwo_detector_free": (None, [C.c_void_p]),
            "cwo_detector_observe": (None, [C.c_void_p, D, dp]),
            "cwo_assemble_slab3d": (D, [I64, I64, I64, D, D, D, dp, C.POINTER(lp), C.POINTER(lp), C.POINTER(dp),
                                        C.POINTER(dp)]),
            "cwo_free": (None, [C.c_void_p]),
            "cwo_reaction_step_omp": (I64, [I64, I, dp, dp, dp, u8p, ip, ip, dp, C.c_void_p, I, I, I, D, D, lp, I,
                                            dp]),
            "cwo_slab3d_classes": (D, [I64, D, D, D, dp, dp, dp]),
            "cwo_diffusion_substep_slab3d": (None, [I64, I64, I64, dp, dp, dp, D, dp]),
            "cwo_mt64_raw": (None, [C.c_uint64, I64, C.POINTER(C.c_uint64)]),
            "cwo_uniform_mt64": (None, [C.c_uint64, I64, D, D, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _lp(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def state_count(model):
    return lib().cwo_state_count(MODEL_KINDS[model])


def stable_step(model):
    return lib().cwo_stable_step(MODEL_KINDS[model])


def rest_state(model):
    out = np.zeros(64)
    lib().cwo_rest_state(MODEL_KINDS[model], _dp(out))
    return out[: state_count(model) + 1].copy()


def rates(model, v, s, i_stim):
    v = np.ascontiguousarray(v, np.float64)
    s = np.ascontiguousarray(s, np.float64)
    i_stim = np.ascontiguousarray(i_stim, np.float64)
    dv = np.zeros(v.shape[0])
    ds = np.zeros_like(s)
    lib().cwo_rates_batch(MODEL_KINDS[model], v.shape[0], _dp(v), _dp(s), _dp(i_stim), _dp(dv), _dp(ds))
    return dv, ds


def pace(model, cycle_ms, n_beats, amp, dur):
    """pace_to_steady_state restatement (ionic.cpp:122-165): (state, max_rel, apd90[n_beats]);
    raises OracleInstability(msg, -1, t) on divergence, ValueError on bad arguments."""
    st = np.zeros(64)
    apd = np.zeros(max(1, n_beats))
    mr = C.c_double()
    fb = C.c_int()
    ft = C.c_double()
    rc = lib().cwo_pace(MODEL_KINDS[model], cycle_ms, n_beats, amp, dur, _dp(st), _dp(apd), C.byref(mr),
                        C.byref(fb), C.byref(ft))
    if rc == 1:
        raise ValueError("pacing: invalid arguments")
    if rc in (2, 3):
        raise OracleInstability(f"pacing: diverged at beat {fb.value}", -1, ft.value)
    return st[: state_count(model) + 1].copy(), mr.value, apd[:n_beats].copy()


def reaction_substeps(dvdt, scheme, k0_up, k0_down, k_max):
    return lib().cwo_reaction_substeps(float(dvdt), SCHEMES[scheme], k0_up, k0_down, k_max)


def diffusion_substeps(dt, dt_s, strict, scheme):
    l, dt_ad = C.c_int(), C.c_double()
    rc = lib().cwo_diffusion_substeps(dt, dt_s, int(strict), SCHEMES[scheme], C.byref(l), C.byref(dt_ad))
    if rc:
        raise ValueError("diffusion sub-steps: dt and dt_s must be positive")
    return l.value, dt_ad.value


def k_max_for(dt, model):
    return lib().cwo_k_max_for(dt, stable_step(model))


def assemble_slab3d(nx, ny, nz, h, d_long, rho, angles):
    """CSR (row_ptr, col, val, mass) and dt_s of the 3D slab operator (extension)."""
    L = lib()
    ang = np.ascontiguousarray(angles, np.float64)
    rp, col, val, mass = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
    dt_s = L.cwo_assemble_slab3d(nx, ny, nz, h, d_long, rho, _dp(ang), C.byref(rp), C.byref(col), C.byref(val),
                                 C.byref(mass))
    n = (nx + 1) * (ny + 1) * (nz + 1)
    rpa = np.ctypeslib.as_array(rp, (n + 1,)).copy()
    nnz = int(rpa[-1])
    out = (rpa, np.ctypeslib.as_array(col, (nnz,)).copy(), np.ctypeslib.as_array(val, (nnz,)).copy(),
           np.ctypeslib.as_array(mass, (n,)).copy())
    for ptr in (rp, col, val, mass):
        L.cwo_free(C.cast(ptr, C.c_void_p))
    return out, dt_s


def mt64_raw(seed, n):
    out = np.zeros(n, np.uint64)
    lib().cwo_mt64_raw(seed, n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def uniform_mt64(seed, n, lo, hi):
    out = np.zeros(n)
    lib().cwo_uniform_mt64(seed, n, lo, hi, _dp(out))
    return out


class Slab3DOp:
    """Structured 3D slab operator (EXTENSION, BASELINE configs 4-5) for the oracle run loop: node-class
    tables from the oracle's own CSR assembly of a 2 x 2 x nz-element slab (cwo_slab3d_classes), applied
    matrix-free (cwo_diffusion_substep_slab3d), so 10^6-10^8-node slabs need no CSR. Node index
    (iy*(nz+1) + iz)*(nx+1) + ix; fibre angle per element layer linear in z (endo -> epi)."""

    def __init__(self, nx, ny, nz, h, d_long=0.0012, rho=0.25, angle_endo_deg=60.0, angle_epi_deg=-60.0):
        self.nx, self.ny, self.nz, self.h = nx, ny, nz, h
        self.nx1, self.ny1, self.nz1 = nx + 1, ny + 1, nz + 1
        self.n = self.nx1 * self.ny1 * self.nz1
        self.angles = np.deg2rad(angle_endo_deg + (angle_epi_deg - angle_endo_deg) * (np.arange(nz) + 0.5) / nz)
        self.coef = np.zeros(9 * self.nz1 * 27)
        self.mass = np.zeros(9 * self.nz1)
        self.dt_s = lib().cwo_slab3d_classes(nz, h, d_long, rho, _dp(self.angles), _dp(self.coef), _dp(self.mass))

    def index(self, ix, iy, iz):
        return (np.asarray(iy) * self.nz1 + np.asarray(iz)) * self.nx1 + np.asarray(ix)

    def substep(self, v, dt_sub):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty_like(v)
        lib().cwo_diffusion_substep_slab3d(self.nx1, self.ny1, self.nz1, _dp(self.coef), _dp(self.mass), _dp(v),
                                           dt_sub, _dp(out))
        return out


def diffusion_substep(csr, v, dt_sub):
    if hasattr(csr, "substep"):
        return csr.substep(v, dt_sub)
    rp, col, val, mass = csr
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty_like(v)
    lib().cwo_diffusion_substep_csr(len(mass), _lp(rp), _lp(col), _dp(val), _dp(mass), _dp(v), dt_sub, _dp(out))
    return out


class _Prot(C.Structure):
    _fields_ = [("node_ptr", C.POINTER(C.c_int32)), ("ids", C.POINTER(C.c_int32)),
                ("t_start", C.POINTER(C.c_double)), ("duration", C.POINTER(C.c_double)),
                ("amplitude", C.POINTER(C.c_double)), ("period", C.POINTER(C.c_double))]


class Protocol:
    """Flattened ProtocolIndex (stimulus.cpp:17-31): per-node entry-id lists."""

    def __init__(self, n, stimuli):
        # stimuli: list of (nodes, t_start, duration, amplitude, period|None)
        # per node, entry ids in entry order (stimulus.cpp:17-31 appends entry by entry)
        nodes = [np.asarray(st[0], np.int64).ravel() for st in stimuli]
        eids = [np.full(len(nd), e, np.int32) for e, nd in enumerate(nodes)]
        nd = np.concatenate(nodes) if nodes else np.zeros(0, np.int64)
        ed = np.concatenate(eids) if eids else np.zeros(0, np.int32)
        order = np.argsort(nd, kind="stable")
        self.node_ptr = np.zeros(n + 1, np.int32)
        self.node_ptr[1:] = np.cumsum(np.bincount(nd, minlength=n)[:n])
        self.ids = ed[order].astype(np.int32) if ed.size else np.array([0], np.int32)
        self.t_start = np.array([s[1] for s in stimuli] or [0.0])
        self.duration = np.array([s[2] for s in stimuli] or [0.0])
        self.amplitude = np.array([s[3] for s in stimuli] or [0.0])
        self.period = np.array([math.nan if s[4] is None else s[4] for s in stimuli] or [math.nan])
        i32 = C.POINTER(C.c_int32)
        self.c = _Prot(self.node_ptr.ctypes.data_as(i32), self.ids.ctypes.data_as(i32), _dp(self.t_start),
                       _dp(self.duration), _dp(self.amplitude), _dp(self.period))

    def current(self, node, t):
        return lib().cwo_stim_current(C.byref(self.c), node, t)


class _Det(C.Structure):
    _fields_ = [("n", C.c_int64), ("threshold", C.c_double), ("prev_t", C.c_double), ("first", C.c_int)] + \
        [(nm, C.POINTER(C.c_double)) for nm in ("prev_v", "v_rest", "max_slope", "t_max_slope", "v_peak", "lat", "apd")] + \
        [(nm, C.POINTER(C.c_uint8)) for nm in ("phase", "has_lat", "has_apd")]


class Detector:
    def __init__(self, n, threshold=0.0):
        self.n = n
        self.d = _Det()
        lib().cwo_detector_init(C.byref(self.d), n, threshold)

    def observe(self, t, v):
        v = np.ascontiguousarray(v, np.float64)
        lib().cwo_detector_observe(C.byref(self.d), t, _dp(v))

    def maps(self):
        n = self.n
        def arr(p, dt):
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt).copy()
        lat = arr(self.d.lat, np.float64)
        apd = arr(self.d.apd, np.float64)
        lv = arr(self.d.has_lat, bool)
        av = arr(self.d.has_apd, bool)
        lat[~lv] = np.nan
        apd[~av] = np.nan
        return lat, lv, apd, av

    def __del__(self):
        if _lib is not None:
            _lib.cwo_detector_free(C.byref(self.d))


class OracleInstability(RuntimeError):
    def __init__(self, msg, node, t):
        super().__init__(f"{msg} (node {node}, t = {t:.6f} ms)")
        self.node, self.t = node, t


def run_simulation(csr, dt_s, models, model_of_node, stimuli, scheme="DAETI", dt=0.1, t_end=1.0, k0_up=5,
                   k0_down=1, strict=False, record_interval=1.0, map_interval=1.0, probes=(), lat_threshold=0.0,
                   init=None, gkr_scale=None, stride=None, snapshot_interval=0.0):
    """Restatement of run_simulation (splitting.cpp:219-294) + StrangIntegrator (:74-181).

    models: list of model names (model id -> name); model_of_node: uint8[n].
    stimuli: list of (nodes, t_start, duration, amplitude, period|None).
    init: optional (v, s_aos[n, stride], last_dvdt) to start from.
    Raises OracleInstability like the reference's InstabilityError.
    """
    L = lib()
    n = csr.n if hasattr(csr, "substep") else len(csr[3])
    kinds = np.array([MODEL_KINDS[m] for m in models], np.int32)
    sc = SCHEMES[scheme]
    dt_eff = min(dt, dt_s) if scheme == "OSTAR" else dt
    l, dt_ad = diffusion_substeps(dt_eff, dt_s, strict, scheme)
    kmax = np.array([max(1, int(math.floor(dt_eff / stable_step(m)))) for m in models], np.int32)
    kmax_g = max(1, int(kmax.max()))
    if stride is None:
        stride = max([1] + [state_count(m) for m in models])
    model_of_node = np.ascontiguousarray(model_of_node, np.uint8)
    if init is None:
        v = np.zeros(n)
        s = np.zeros((n, stride))
        last = np.zeros(n)
        for mid, m in enumerate(models):
            r = rest_state(m)
            sel = model_of_node == mid
            v[sel] = r[0]
            s[np.ix_(sel, np.arange(len(r) - 1))] = r[1:]
    else:
        v, s, last = (np.array(a, np.float64, copy=True) for a in init)
        s = s.reshape(n, stride)
    s = np.ascontiguousarray(s)
    prot = Protocol(n, stimuli)
    khist = np.zeros(kmax_g + 1, np.int64)
    gk = None if gkr_scale is None else np.ascontiguousarray(gkr_scale, np.float64)
    n_steps = int(math.ceil(t_end / dt_eff - 1e-9))
    spr = max(1, int(round_half_away(record_interval / dt_eff)))
    spm = max(1, int(round_half_away(map_interval / dt_eff)))
    det = Detector(n, lat_threshold)
    sps = max(1, int(round_half_away(snapshot_interval / dt_eff))) if snapshot_interval > 0.0 else 0
    snaps = [(0.0, v.copy())] if sps else []
    traces_t = [0.0]
    traces_v = [[float(v[p]) for p in probes]]
    det.observe(0.0, v)
    bad_t = C.c_double()
    u8p = C.POINTER(C.c_uint8)
    ip = C.POINTER(C.c_int)

    def diffuse(count, t):
        nonlocal v
        for _ in range(count):
            v = diffusion_substep(csr, v, dt_ad)
            bad = np.flatnonzero(~np.isfinite(v))
            if bad.size:
                raise OracleInstability("diffusion sub-step produced non-finite V", int(bad[0]), t)

    for step in range(n_steps):
        t = float(step) * dt_eff
        if step == 0:
            diffuse(l, t)
        bad = L.cwo_reaction_step_omp(n, stride, _dp(v), _dp(s), _dp(last), model_of_node.ctypes.data_as(u8p),
                                      kinds.ctypes.data_as(ip), kmax.ctypes.data_as(ip),
                                      None if gk is None else _dp(gk), C.byref(prot.c), sc, k0_up, k0_down,
                                      dt_eff, t, _lp(khist), len(khist), C.byref(bad_t))
        if bad >= 0:
            raise OracleInstability("reaction step produced non-finite V", int(bad), bad_t.value)
        diffuse(l if step == n_steps - 1 else 2 * l, t)
        t_next = float(step + 1) * dt_eff
        if (step + 1) % spr == 0:
            traces_t.append(t_next)
            traces_v.append([float(v[p]) for p in probes])
        if (step + 1) % spm == 0:
            det.observe(t_next, v)
        if sps and (step + 1) % sps == 0:  # on_snapshot (splitting.cpp:276-277)
            snaps.append((t_next, v.copy()))
    lat, lv, apd, av = det.maps()
    return dict(v=v, s=s, last_dvdt=last, k_histogram=khist, n_steps=n_steps, l=l, dt_ad=dt_ad, snapshots=snaps,
                dt_effective=dt_eff, trace_t=np.array(traces_t), traces=np.array(traces_v).T.copy(),
                lat=lat, lat_valid=lv, apd90=apd, apd_valid=av)


class Integrator:
    """StrangIntegrator restatement with the reference's per-step surface (splitting.hpp:101-127):
    advance(t, step, n_steps) runs splitting.cpp:171-181 on the oracle kernels (OpenMP reaction and
    diffusion). Used by bench.py's CPU legs on configurations the reference cannot express."""

    def __init__(self, op, dt_s, models, model_of_node, stimuli, scheme="DAETI", dt=0.1, k0_up=5, k0_down=1,
                 strict=False, gkr_scale=None):
        self.op = op
        self.n = op.n if hasattr(op, "substep") else len(op[3])
        self.kinds = np.array([MODEL_KINDS[m] for m in models], np.int32)
        self.sc = SCHEMES[scheme]
        self.dt_eff = min(dt, dt_s) if scheme == "OSTAR" else dt
        self.l, self.dt_ad = diffusion_substeps(self.dt_eff, dt_s, strict, scheme)
        self.kmax = np.array([max(1, int(math.floor(self.dt_eff / stable_step(m)))) for m in models], np.int32)
        self.khist = np.zeros(max(1, int(self.kmax.max())) + 1, np.int64)
        self.stride = max([1] + [state_count(m) for m in models])
        self.mon = np.ascontiguousarray(model_of_node, np.uint8)
        self.k0_up, self.k0_down = k0_up, k0_down
        self.gk = None if gkr_scale is None else np.ascontiguousarray(gkr_scale, np.float64)
        self.prot = Protocol(self.n, stimuli)
        self.v = np.zeros(self.n)
        self.s = np.zeros((self.n, self.stride))
        self.last = np.zeros(self.n)
        for mid, m in enumerate(models):  # make_initial_state (splitting.cpp:183-217), rest states
            r = rest_state(m)
            sel = self.mon == mid
            self.v[sel] = r[0]
            self.s[np.ix_(sel, np.arange(len(r) - 1))] = r[1:]

    def _diffuse(self, count, t):
        for _ in range(count):
            self.v = diffusion_substep(self.op, self.v, self.dt_ad)
            bad = np.flatnonzero(~np.isfinite(self.v))
            if bad.size:
                raise OracleInstability("diffusion sub-step produced non-finite V", int(bad[0]), t)

    def advance(self, t, step, n_steps):
        if step == 0:
            self._diffuse(self.l, t)
        bad_t = C.c_double()
        bad = lib().cwo_reaction_step_omp(self.n, self.stride, _dp(self.v), _dp(self.s), _dp(self.last),
                                          self.mon.ctypes.data_as(C.POINTER(C.c_uint8)),
                                          self.kinds.ctypes.data_as(C.POINTER(C.c_int)),
                                          self.kmax.ctypes.data_as(C.POINTER(C.c_int)),
                                          None if self.gk is None else _dp(self.gk), C.byref(self.prot.c), self.sc,
                                          self.k0_up, self.k0_down, self.dt_eff, t, _lp(self.khist),
                                          len(self.khist), C.byref(bad_t))
        if bad >= 0:
            raise OracleInstability("reaction step produced non-finite V", int(bad), bad_t.value)
        self._diffuse(self.l if step == n_steps - 1 else 2 * self.l, t)


def round_half_away(x):
    """std::llround semantics (half away from zero)."""
    return math.floor(x + 0.5) if x >= 0 else -math.floor(-x + 0.5)
