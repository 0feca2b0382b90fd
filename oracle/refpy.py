"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libcwref.so.

libcwref.so is the *unmodified* reference library (cardwave, built from
/root/reference/proj/core/src by oracle/Makefile) plus our marshalling shim
oracle/ref_capi.cpp. Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs may import this module; the product path never
does.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcwref.so")

SCHEMES = {"OST": 0, "OSTAR": 1, "DAETI": 2}
REGION_KINDS = {"x_le": 0, "x_ge": 1, "y_le": 2, "y_ge": 3, "rectangle": 4, "node_set": 5, "disc": 6}

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        P, D, I64, I, CP = C.c_void_p, C.c_double, C.c_int64, C.c_int, C.c_char_p
        dp, lp = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        sig = {
            "cwref_sheet": (P, [D, D, D, D, D, D, D, D, C.c_uint64, CP, I]),
            "cwref_free": (None, [P]),
            "cwref_n": (I64, [P]),
            "cwref_nnz": (I64, [P]),
            "cwref_dt_s": (D, [P]),
            "cwref_n_tags": (I, [P]),
            "cwref_csr": (None, [P, lp, lp, dp, dp]),
            "cwref_node_tags": (None, [P, C.POINTER(C.c_int32)]),
            "cwref_tag_name": (None, [P, I, CP, I]),
            "cwref_select": (I64, [P, I, dp, lp, I64, lp, I64]),
            "cwref_nearest": (I64, [P, D, D]),
            "cwref_set_models": (I, [P, C.POINTER(CP), I, CP, I]),
            "cwref_add_stimulus": (I, [P, lp, I64, D, D, D, D]),
            "cwref_clear_stimuli": (None, [P]),
            "cwref_state_stride": (I, [P]),
            "cwref_init_state": (I, [P, CP, I]),
            "cwref_get_state": (None, [P, dp, dp, dp, C.POINTER(C.c_uint8)]),
            "cwref_put_state": (None, [P, dp, dp, dp]),
            "cwref_diffusion_substep": (None, [P, dp, D, dp]),
            "cwref_integrator": (I, [P, I, D, D, I, I, I, I, CP, I]),
            "cwref_advance": (I, [P, D, I64, I64, lp, dp, CP, I]),
            "cwref_integrator_info": (None, [P, dp, C.POINTER(I), dp, C.POINTER(I), dp]),
            "cwref_integrator_khist": (None, [P, lp]),
            "cwref_run": (I, [P, I, D, D, I, I, I, D, I, lp, I, D, CP, I]),
            "cwref_run_error": (None, [P, lp, dp]),
            "cwref_res_n_steps": (I64, [P]),
            "cwref_res_khist_len": (I, [P]),
            "cwref_res_khist": (None, [P, lp]),
            "cwref_res_plan": (None, [P, dp, dp, C.POINTER(I), dp]),
            "cwref_res_timing": (None, [P, dp]),
            "cwref_res_n_samples": (I64, [P]),
            "cwref_res_trace": (None, [P, I, dp, dp]),
            "cwref_res_maps": (None, [P, dp, CP, dp, CP]),
            "cwref_model_info": (I, [CP, C.POINTER(I), dp, dp, I]),
            "cwref_rates": (I, [CP, I64, dp, dp, dp, dp, dp]),
            "cwref_compute_apd90": (I, [dp, dp, I64, dp]),
            "cwref_compute_cv": (I, [C.c_void_p, dp, C.c_char_p, I64, I64, dp]),
            "cwref_nrmse": (I, [I64, dp, C.c_char_p, dp, C.c_char_p, dp]),
            "cwref_align_and_diff": (I, [dp, dp, I64, dp, dp, I64, dp]),
            "cwref_write_vtk_snapshot": (I, [C.c_void_p, dp, C.c_double, CP]),
            "cwref_write_map": (I, [C.c_void_p, dp, C.c_char_p, CP, I, CP]),
            "cwref_write_trace_csv": (I, [dp, dp, I64, CP]),
            "cwref_state_save": (I, [I64, I, dp, dp, dp, C.c_char_p, CP]),
            "cwref_pace": (I, [CP, C.c_double, I, C.c_double, C.c_double, dp, dp, dp, dp, C.c_char_p, I]),
            "cwref_estimate_dt0": (D, [CP]),
            "cwref_reaction_substeps": (I, [D, I, I, I, I]),
            "cwref_diffusion_substeps": (I, [D, D, I, I, C.POINTER(I), dp]),
            "cwref_k_max_for": (I, [D, CP]),
            "cwref_gershgorin": (D, [P]),
            "cwref_threshold": (D, [P, CP, lp, I64, D, D, D, CP, I]),
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


class RefError(RuntimeError):
    def __init__(self, code, msg, node=-1, t=0.0):
        super().__init__(msg)
        self.code, self.node, self.t = code, node, t


def model_info(name: str):
    L = lib()
    ns, ss = C.c_int(), C.c_double()
    rest = np.zeros(64)
    if L.cwref_model_info(name.encode(), C.byref(ns), C.byref(ss), _dp(rest), 64) != 0:
        raise RefError(2, f"unknown model {name}")
    return ns.value, ss.value, rest[: ns.value + 1].copy()


def rates(name: str, v, s, i_stim):
    """Batched CellModel::rates. v[n], s[n, ns], i_stim[n] -> (dv[n], ds[n, ns])."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    i_stim = np.ascontiguousarray(i_stim, dtype=np.float64)
    n = v.shape[0]
    dv = np.zeros(n)
    ds = np.zeros_like(s)
    if lib().cwref_rates(name.encode(), n, _dp(v), _dp(s), _dp(i_stim), _dp(dv), _dp(ds)) != 0:
        raise RefError(2, f"unknown model {name}")
    return dv, ds


def compute_apd90(t, v):
    t, v = np.ascontiguousarray(t, np.float64), np.ascontiguousarray(v, np.float64)
    out = C.c_double()
    return out.value if lib().cwref_compute_apd90(_dp(t), _dp(v), len(t), C.byref(out)) else None


def _u8(a):
    return np.ascontiguousarray(a, np.uint8).tobytes()


def compute_cv(sheet, lat, valid, a, b):
    lat = np.ascontiguousarray(lat, np.float64)
    out = C.c_double()
    if lib().cwref_compute_cv(sheet.p, _dp(lat), _u8(valid), a, b, C.byref(out)) != 0:
        raise RefError(2, "compute_cv: validation error")
    return out.value


def nrmse(rv, rvalid, cv, cvalid):
    rv, cv = np.ascontiguousarray(rv, np.float64), np.ascontiguousarray(cv, np.float64)
    out = C.c_double()
    if lib().cwref_nrmse(len(rv), _dp(rv), _u8(rvalid), _dp(cv), _u8(cvalid), C.byref(out)) != 0:
        raise RefError(2, "nrmse: validation error")
    return out.value


def align_and_diff(ta, va, tb, vb):
    ta, va, tb, vb = (np.ascontiguousarray(x, np.float64) for x in (ta, va, tb, vb))
    out = C.c_double()
    if lib().cwref_align_and_diff(_dp(ta), _dp(va), len(ta), _dp(tb), _dp(vb), len(tb), C.byref(out)) != 0:
        raise RefError(2, "align: validation error")
    return out.value


def write_vtk_snapshot(sheet, v, t, path):
    v = np.ascontiguousarray(v, np.float64)
    assert lib().cwref_write_vtk_snapshot(sheet.p, _dp(v), t, path.encode()) == 0


def write_map(sheet, value, valid, name, vtk, path):
    value = np.ascontiguousarray(value, np.float64)
    assert lib().cwref_write_map(sheet.p, _dp(value), _u8(valid), name.encode(), int(vtk), path.encode()) == 0


def write_trace_csv(t, v, path):
    t, v = np.ascontiguousarray(t, np.float64), np.ascontiguousarray(v, np.float64)
    assert lib().cwref_write_trace_csv(_dp(t), _dp(v), len(t), path.encode()) == 0


def state_save(n, stride, v, s, last, mon, path):
    v, s, last = (np.ascontiguousarray(x, np.float64) for x in (v, s, last))
    assert lib().cwref_state_save(n, stride, _dp(v), _dp(s), _dp(last), _u8(mon), path.encode()) == 0


def pace(name, cycle_ms, n_beats, amp, dur):
    """cardwave::pace_to_steady_state: (state, max_rel_change, apd90[n_beats])."""
    st = np.zeros(64)
    apd = np.zeros(max(1, n_beats))
    mr, ft = C.c_double(), C.c_double()
    msg = C.create_string_buffer(256)
    rc = lib().cwref_pace(name.encode(), cycle_ms, n_beats, amp, dur, _dp(st), _dp(apd), C.byref(mr), C.byref(ft),
                          msg, 256)
    if rc != 0:
        raise RefError(rc, msg.value.decode(), -1, ft.value)
    ns = model_info(name)[0]
    return st[: ns + 1].copy(), mr.value, apd[:n_beats].copy()


def reaction_substeps(dvdt, scheme, k0_up, k0_down, k_max):
    return lib().cwref_reaction_substeps(float(dvdt), SCHEMES[scheme], k0_up, k0_down, k_max)


def diffusion_substeps(dt, dt_s, strict, scheme):
    l, dt_ad = C.c_int(), C.c_double()
    rc = lib().cwref_diffusion_substeps(dt, dt_s, int(strict), SCHEMES[scheme], C.byref(l), C.byref(dt_ad))
    if rc != 0:
        raise RefError(rc, "diffusion_substeps rejected")
    return l.value, dt_ad.value


def k_max_for(dt, model):
    return lib().cwref_k_max_for(dt, model.encode())


class Sheet:
    """A reference problem: regular sheet + assembled operator + models + protocol."""

    def __init__(self, lx, ly, h, angle_rad=0.0, d0=0.0017, d0_fib=0.00066, rho=0.25,
                 fib_fraction=0.0, seed=0):
        L = lib()
        err = C.create_string_buffer(512)
        self.p = L.cwref_sheet(lx, ly, h, angle_rad, d0, d0_fib, rho, fib_fraction, seed, err, 512)
        if not self.p:
            raise RefError(2, err.value.decode())
        self.n = L.cwref_n(self.p)
        self.nnz = L.cwref_nnz(self.p)
        self.dt_s = L.cwref_dt_s(self.p)
        self.nx1 = int(round(lx / h)) + 1

    def __del__(self):
        if getattr(self, "p", None) and _lib is not None:
            _lib.cwref_free(self.p)
            self.p = None

    def csr(self):
        rp = np.zeros(self.n + 1, np.int64)
        col = np.zeros(self.nnz, np.int64)
        val = np.zeros(self.nnz)
        mass = np.zeros(self.n)
        lib().cwref_csr(self.p, _lp(rp), _lp(col), _dp(val), _dp(mass))
        return rp, col, val, mass

    def tags(self):
        t = np.zeros(self.n, np.int32)
        lib().cwref_node_tags(self.p, t.ctypes.data_as(C.POINTER(C.c_int32)))
        names = []
        for i in range(lib().cwref_n_tags(self.p)):
            b = C.create_string_buffer(128)
            lib().cwref_tag_name(self.p, i, b, 128)
            names.append(b.value.decode())
        return t, names

    def select(self, kind, value=0.0, x0=0.0, x1=0.0, y0=0.0, y1=0.0, cx=0.0, cy=0.0, radius=0.0,
               nodes=()):
        prm = np.array([value, x0, x1, y0, y1, cx, cy, radius], np.float64)
        sn = np.array(list(nodes), np.int64) if len(nodes) else np.zeros(1, np.int64)
        out = np.zeros(self.n, np.int64)
        m = lib().cwref_select(self.p, REGION_KINDS[kind], _dp(prm), _lp(sn), len(nodes), _lp(out), self.n)
        return out[:m].copy()

    def nearest(self, x, y):
        return lib().cwref_nearest(self.p, x, y)

    def set_models(self, names):
        arr = (C.c_char_p * len(names))(*[n.encode() for n in names])
        err = C.create_string_buffer(512)
        rc = lib().cwref_set_models(self.p, arr, len(names), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())

    def add_stimulus(self, nodes, t0, dur, amp, period=None):
        nodes = np.ascontiguousarray(nodes, np.int64)
        lib().cwref_add_stimulus(self.p, _lp(nodes), len(nodes), t0, dur, amp,
                                 math.nan if period is None else period)

    def init_state(self):
        err = C.create_string_buffer(512)
        rc = lib().cwref_init_state(self.p, err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        self.stride = lib().cwref_state_stride(self.p)

    def get_state(self):
        v = np.zeros(self.n)
        s = np.zeros(self.n * self.stride)
        d = np.zeros(self.n)
        m = np.zeros(self.n, np.uint8)
        lib().cwref_get_state(self.p, _dp(v), _dp(s), _dp(d), m.ctypes.data_as(C.POINTER(C.c_uint8)))
        return v, s.reshape(self.n, self.stride), d, m

    def put_state(self, v=None, s=None, last_dvdt=None):
        def ptr(a):
            return None if a is None else _dp(np.ascontiguousarray(a, np.float64))
        keep = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (v, s, last_dvdt)]
        lib().cwref_put_state(self.p, *[None if a is None else _dp(a) for a in keep])

    def diffusion_substep(self, v, dt_sub):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(self.n)
        lib().cwref_diffusion_substep(self.p, _dp(v), dt_sub, _dp(out))
        return out

    # -- StrangIntegrator, step-wise
    def integrator(self, scheme="DAETI", dt=0.1, t_end=1.0, k0_up=5, k0_down=1, strict=False, workers=0):
        err = C.create_string_buffer(512)
        rc = lib().cwref_integrator(self.p, SCHEMES[scheme], dt, t_end, k0_up, k0_down, int(strict), workers,
                                    err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        dt_eff, l, dt_ad, kmax = C.c_double(), C.c_int(), C.c_double(), C.c_int()
        lib().cwref_integrator_info(self.p, C.byref(dt_eff), C.byref(l), C.byref(dt_ad), C.byref(kmax), None)
        self.dt_eff, self.l, self.dt_ad, self.k_max_global = dt_eff.value, l.value, dt_ad.value, kmax.value

    def advance(self, t, step, n_steps):
        node, tt = C.c_int64(-1), C.c_double(0.0)
        err = C.create_string_buffer(512)
        rc = lib().cwref_advance(self.p, t, step, n_steps, C.byref(node), C.byref(tt), err, 512)
        if rc:
            raise RefError(rc, err.value.decode(), node.value, tt.value)

    def integrator_khist(self):
        h = np.zeros(self.k_max_global + 1, np.int64)
        lib().cwref_integrator_khist(self.p, _lp(h))
        return h

    # -- run_simulation
    def run(self, scheme="DAETI", dt=0.1, t_end=1.0, k0_up=5, k0_down=1, strict=False, record_interval=1.0,
            workers=0, probes=(), lat_threshold=0.0):
        pr = np.array(list(probes), np.int64) if len(probes) else np.zeros(1, np.int64)
        err = C.create_string_buffer(512)
        rc = lib().cwref_run(self.p, SCHEMES[scheme], dt, t_end, k0_up, k0_down, int(strict), record_interval,
                             workers, _lp(pr), len(probes), lat_threshold, err, 512)
        if rc:
            node, tt = C.c_int64(), C.c_double()
            lib().cwref_run_error(self.p, C.byref(node), C.byref(tt))
            raise RefError(rc, err.value.decode(), node.value, tt.value)
        res = {}
        res["n_steps"] = lib().cwref_res_n_steps(self.p)
        kh = np.zeros(lib().cwref_res_khist_len(self.p), np.int64)
        lib().cwref_res_khist(self.p, _lp(kh))
        res["k_histogram"] = kh
        dt_eff, dt_s, l, dt_ad = C.c_double(), C.c_double(), C.c_int(), C.c_double()
        lib().cwref_res_plan(self.p, C.byref(dt_eff), C.byref(dt_s), C.byref(l), C.byref(dt_ad))
        res.update(dt_effective=dt_eff.value, dt_s=dt_s.value, l=l.value, dt_ad=dt_ad.value)
        t4 = np.zeros(4)
        lib().cwref_res_timing(self.p, _dp(t4))
        res["timing_ms"] = dict(total=t4[0], reaction=t4[1], diffusion=t4[2], recording=t4[3])
        ns = lib().cwref_res_n_samples(self.p)
        tr = []
        for q in range(len(probes)):
            t = np.zeros(ns)
            v = np.zeros(ns)
            lib().cwref_res_trace(self.p, q, _dp(t), _dp(v))
            tr.append((t, v))
        res["traces"] = tr
        lat, apd = np.zeros(self.n), np.zeros(self.n)
        lv = C.create_string_buffer(self.n)
        av = C.create_string_buffer(self.n)
        lib().cwref_res_maps(self.p, _dp(lat), lv, _dp(apd), av)
        res["lat"] = lat
        res["lat_valid"] = np.frombuffer(lv.raw, np.uint8).astype(bool)
        res["apd90"] = apd
        res["apd_valid"] = np.frombuffer(av.raw, np.uint8).astype(bool)
        res["state"] = self.get_state()
        return res

    def threshold(self, model, nodes, window_ms=50.0, duration_ms=1.0, initial_guess=1.0):
        nodes = np.ascontiguousarray(nodes, np.int64)
        err = C.create_string_buffer(512)
        r = lib().cwref_threshold(self.p, model.encode(), _lp(nodes), len(nodes), window_ms, duration_ms,
                                  initial_guess, err, 512)
        if math.isnan(r):
            raise RefError(2, err.value.decode())
        return r
