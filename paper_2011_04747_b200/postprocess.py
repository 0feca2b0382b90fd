"""Post-processing metrics of a finished run, restated from the reference's
postprocess.cpp (host-side arithmetic on traces and maps, in the reference's
operation order, so results are bit-identical to cardwave's own functions):

* compute_apd90  (postprocess.cpp:98-134)
* compute_cv     (:136-148)
* nrmse          (:150-168)
* align_and_diff (:172-236, with max_slope_instant and interp)

Plus compare_schemes, the device counterpart of cli_compare
(runner.cpp:254-324): every scheme runs on ONE StrangIntegrator whose
operator stays resident on the GPU (cwg_set_scheme between runs).
"""
import bisect
import ctypes
import ctypes.util
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import api
from .api import ScalarMap, Scheme, SchemeConfig, Trace, ValidationError

K_MIN_AP_AMPLITUDE = 20.0  # mV (postprocess.cpp:12)

_libm = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
_libm.hypot.restype = ctypes.c_double
_libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]


def compute_apd90(trace: Trace) -> Optional[float]:
    """Onset at the maximum finite-difference slope (pair midpoint), V90 from the
    pre-onset minimum and the post-onset peak, linear crossing; None = no AP."""
    t, v = [float(x) for x in trace.t_ms], [float(x) for x in trace.v_mv]
    n = len(t)
    if n < 3:
        return None
    max_slope, slope_idx = -math.inf, 0
    for i in range(n - 1):
        s = (v[i + 1] - v[i]) / (t[i + 1] - t[i])
        if s > max_slope:
            max_slope, slope_idx = s, i
    t_start = 0.5 * (t[slope_idx] + t[slope_idx + 1])
    v_rest = v[0]
    for i in range(slope_idx + 1):
        v_rest = min(v_rest, v[i])
    v_peak, peak_idx = -math.inf, slope_idx
    for i in range(slope_idx, n):
        if v[i] > v_peak:
            v_peak, peak_idx = v[i], i
    if v_peak - v_rest < K_MIN_AP_AMPLITUDE:
        return None
    v90 = v_peak - 0.9 * (v_peak - v_rest)
    for i in range(peak_idx, n - 1):
        if v[i] >= v90 and v[i + 1] < v90:
            frac = (v[i] - v90) / (v[i] - v[i + 1])
            t_cross = t[i] + frac * (t[i + 1] - t[i])
            return t_cross - t_start
    return None


def compute_cv(coords, lat: ScalarMap, probe_a: int, probe_b: int) -> float:
    """Conduction velocity between two probes: |x_a - x_b| / |LAT_b - LAT_a| (cm/ms)."""
    n = len(lat.value)
    if probe_a < 0 or probe_b < 0 or probe_a >= n or probe_b >= n:
        raise ValidationError("compute_cv: probe index out of range")
    if not lat.valid[probe_a] or not lat.valid[probe_b]:
        raise ValidationError("compute_cv: probe never activated")
    dlat = abs(float(lat.value[probe_b]) - float(lat.value[probe_a]))
    if dlat == 0.0:
        raise ValidationError("compute_cv: equal activation times at the probes")
    dx = float(coords[probe_a][0]) - float(coords[probe_b][0])
    dy = float(coords[probe_a][1]) - float(coords[probe_b][1])
    return _libm.hypot(dx, dy) / dlat


def nrmse(reference: ScalarMap, candidate: ScalarMap) -> float:
    """RMS difference over nodes valid in both, normalised by the reference's range."""
    rv, rok = np.asarray(reference.value, np.float64), np.asarray(reference.valid).astype(bool)
    cv, cok = np.asarray(candidate.value, np.float64), np.asarray(candidate.valid).astype(bool)
    if len(rv) != len(cv):
        raise ValidationError("nrmse: maps differ in node count")
    if rok.any():
        u_min, u_max = float(rv[rok].min()), float(rv[rok].max())
    else:
        u_min, u_max = math.inf, -math.inf
    both = rok & cok
    count = int(both.sum())
    if count == 0:
        raise ValidationError("nrmse: no common valid nodes")
    if not u_max > u_min:
        raise ValidationError("nrmse: reference range is zero")
    d = cv[both] - rv[both]
    sq = float(np.cumsum(d * d)[-1])  # sequential accumulation in node order, as the reference loop
    return math.sqrt(sq / float(count)) / (u_max - u_min)


def _max_slope_instant(tr: Trace) -> float:
    t, v = [float(x) for x in tr.t_ms], [float(x) for x in tr.v_mv]
    n = len(t)
    if n < 2:
        raise ValidationError("align: trace too short")
    slope, mid = [0.0] * (n - 1), [0.0] * (n - 1)
    best, bi = -math.inf, 0
    for i in range(n - 1):
        slope[i] = (v[i + 1] - v[i]) / (t[i + 1] - t[i])
        mid[i] = 0.5 * (t[i] + t[i + 1])
        if slope[i] > best:
            best, bi = slope[i], i
    if best < K_MIN_AP_AMPLITUDE / 10.0:
        raise ValidationError("align: no action potential detected in trace")
    if bi == 0 or bi + 1 >= len(slope):
        return mid[bi]
    y0, y1, y2 = slope[bi - 1], slope[bi], slope[bi + 1]
    den = y0 - 2.0 * y1 + y2
    if den >= 0.0:
        return mid[bi]
    delta = 0.5 * (y0 - y2) / den
    h = mid[bi + 1] - mid[bi]
    return mid[bi] + min(max(delta, -1.0), 1.0) * h


def _interp(t, v, x: float) -> float:
    i = bisect.bisect_right(t, x)
    if i == 0 or i == len(t):
        raise ValidationError("align: interpolation outside trace support")
    i -= 1
    f = (x - t[i]) / (t[i + 1] - t[i])
    return v[i] + f * (v[i + 1] - v[i])


def align_and_diff(trace_a: Trace, trace_b: Trace) -> float:
    """Max |dV| after aligning the two upstrokes (coarser grid, finer trace interpolated)."""
    ta, tb = _max_slope_instant(trace_a), _max_slope_instant(trace_b)
    shift = tb - ta

    def interval(tr):
        return float(tr.t_ms[1]) - float(tr.t_ms[0]) if len(tr.t_ms) > 1 else 0.0

    a_coarse = interval(trace_a) >= interval(trace_b)
    coarse, fine = (trace_a, trace_b) if a_coarse else (trace_b, trace_a)
    to_fine = shift if a_coarse else -shift
    ft, fv = [float(x) for x in fine.t_ms], [float(x) for x in fine.v_mv]
    max_diff, anyp = 0.0, False
    for tc, vc in zip(coarse.t_ms, coarse.v_mv):
        tf = float(tc) + to_fine
        if tf <= ft[0] or tf >= ft[-1]:
            continue
        max_diff = max(max_diff, abs(float(vc) - _interp(ft, fv, tf)))
        anyp = True
    if not anyp:
        raise ValidationError("align: traces do not overlap after alignment")
    return max_diff


# ----------------------------------------------------------------------------- cli_compare
@dataclass
class SchemeComparison:
    """runner.hpp:66-76."""
    scheme: str
    cv_cm_per_ms: float = math.nan
    apd90_per_probe: List[float] = field(default_factory=list)
    wall_ms: float = 0.0
    reaction_ms: float = 0.0
    diffusion_ms: float = 0.0
    e_lat: float = 0.0
    e_apd: float = 0.0
    max_dv_per_probe: List[float] = field(default_factory=list)
    result: object = None  # the scheme's SimulationResult


@dataclass
class CompareReport:
    reference: str
    schemes: List[SchemeComparison]


def compare_schemes(state, setup, cfg: SchemeConfig, coords, schemes: Sequence[str] = ("OST", "OSTAR", "DAETI"),
                    reference: Optional[str] = None, model_of_node=None, device=0) -> CompareReport:
    """cli_compare (runner.cpp:254-324) with one device-resident operator.

    Each scheme runs from the same initial state with the conventional step
    (0.01 ms for OST, 0.1 ms for OSTAR / DAETI; OSTAR then drops to dt_s);
    the integrator is created once and reconfigured with cwg_set_scheme.
    Metrics as the reference: CV between the first two probes (NaN when
    unsuitable), APD90 per probe trace, and against the reference scheme
    NRMSE of the LAT / APD90 maps and the aligned max |dV| per probe."""
    if len(schemes) < 2:
        raise ValidationError("compare: need at least two schemes")
    ref_name = reference if reference in schemes else schemes[0]
    integ = None
    runs = []
    try:
        for name in schemes:
            sch = api.scheme_from_string(name)
            sc = SchemeConfig(scheme=sch, dt_ms=0.01 if sch == Scheme.OST else 0.1, t_end_ms=cfg.t_end_ms,
                              k0_up=cfg.k0_up, k0_down=cfg.k0_down, strict_substeps=cfg.strict_substeps,
                              record_interval_ms=cfg.record_interval_ms)
            if integ is None:
                integ = api.StrangIntegrator(setup, sc, model_of_node=model_of_node, device=device)
            else:
                integ.set_scheme(sc)
            runs.append((name, api.run_simulation(state.copy(), setup, sc, device=device, integrator=integ)))
    finally:
        if integ is not None:
            integ.close()
    ref = dict(runs)[ref_name]
    out = []
    for name, r in runs:
        c = SchemeComparison(scheme=name, wall_ms=r.timing.total_ms, reaction_ms=r.timing.reaction_ms,
                             diffusion_ms=r.timing.diffusion_ms, result=r)
        if len(setup.probes) >= 2:
            try:
                c.cv_cm_per_ms = compute_cv(coords, r.lat_map, setup.probes[0].node, setup.probes[1].node)
            except ValidationError:
                c.cv_cm_per_ms = math.nan
        for tr in r.traces:
            a = compute_apd90(tr)
            c.apd90_per_probe.append(math.nan if a is None else a)
        if r is not ref:
            c.e_lat = nrmse(ref.lat_map, r.lat_map)
            c.e_apd = nrmse(ref.apd90_map, r.apd90_map)
            c.max_dv_per_probe = [align_and_diff(ref.traces[p], r.traces[p]) for p in range(len(r.traces))]
        else:
            c.max_dv_per_probe = [0.0] * len(r.traces)
        out.append(c)
    return CompareReport(ref_name, out)
