"""BASELINE.json configurations as synthetic problems.

There is no public dataset: each config is a seeded synthetic tissue with the
BASELINE shapes. C1/C2 are expressible in the reference as-is (parity pinned
against the reference); C3 needs the extensions (scar with zero
conductivity, passive non-excitable nodes, per-node GKr jitter) and its
parity is pinned only against our CPU restatement oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from . import api


def uniform_mt64(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """n seeded uniform draws in [lo, hi) from std::mt19937_64(seed) (the reference's RNG, mesh.cpp:112):
    lo + (hi - lo) * ((x >> 11) * 2^-53) (cwgpu_setup.h cwg_uniform_mt64)."""
    out = np.zeros(int(n))
    L.lib().cwg_uniform_mt64(int(seed), int(n), float(lo), float(hi), L.dp(out))
    return out


@dataclass
class Problem:
    name: str
    sheet: api.Sheet
    models: List[str]
    model_of_node: np.ndarray
    stimuli: List[tuple]  # (nodes, t_start, duration, amplitude, period|None)
    cfg: api.SchemeConfig
    probes: List[int] = field(default_factory=list)
    gkr_scale: Optional[np.ndarray] = None
    notes: str = ""
    # (model id, cycle length ms, beats, amplitude mV/ms, duration ms): that model's nodes start from
    # pace_to_steady_state (ionic.cpp:122-167) instead of the rest state (computed on the device)
    pacing: Optional[tuple] = None

    @property
    def n(self):
        return self.sheet.n

    def setup(self) -> api.SimulationSetup:
        prot = api.Protocol([api.Stimulus(np.asarray(s[0], np.int64), s[1], s[2], s[3], s[4]) for s in self.stimuli])
        return api.SimulationSetup(op=self.sheet.op, models=[api.make_model(m) for m in self.models],
                                   protocol=api.ProtocolIndex(prot, self.n),
                                   probes=[api.Probe(int(p), f"p{q}") for q, p in enumerate(self.probes)],
                                   gkr_scale=self.gkr_scale)

    def initial_state(self, paced_state=None) -> api.NodeStateArray:
        """make_initial_state; with `pacing`, the paced model's nodes start from its paced state
        (`paced_state` if given, e.g. a fixture's, else pace_to_steady_state on the device)."""
        models = [api.make_model(m) for m in self.models]
        per_model = None
        if self.pacing is not None:
            mid, cl, beats, amp, dur = self.pacing
            if paced_state is None:
                paced_state = api.pace_to_steady_state(models[mid], cl, beats, amp, dur).state
            per_model = [None] * len(models)
            per_model[mid] = np.asarray(paced_state, np.float64)
        return api.make_initial_state(self.n, models, self.model_of_node, initial_per_model=per_model)


# C1: 1x1 cm, h = 0.01, D = 0.001 isotropic; ORd-epi; left-edge line x <= 0 for
# t in [0, 1) at 2 x the reference's diastolic threshold (296 mV/ms, measured
# in the survey with cardwave::diastolic_threshold) = 592 mV/ms; DAETI dt 0.1,
# k0_down = 3 (the paper's k0_down = 1 aborts in the reference).
C1_AMPLITUDE = 592.0
# C2: 5x5 cm, h = 0.025, fibres 45 deg, D_l = 0.0012, D_t = 0.0003; corner disc
# (radius 2h) stimulus. Amplitude chosen stable + propagating in the reference
# (SURVEY.md 8(d) caution 2; probe recorded in DESIGN.md).
C2_AMPLITUDE = 100.0
C2_RADIUS = 0.15


def c1(model="ohara2011-epi", t_end=400.0, k0_down=3, amplitude=None, strip=None, scheme=api.Scheme.DAETI,
       dt=0.1) -> Problem:
    sh = api.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0)
    if model == "aliev-panfilov":
        strip = 0.05 if strip is None else strip
        amplitude = 100.0 if amplitude is None else amplitude
    amp = C1_AMPLITUDE if amplitude is None else amplitude
    nodes = sh.select("x_le", value=0.0 if strip is None else strip)
    cfg = api.SchemeConfig(scheme=scheme, dt_ms=dt, t_end_ms=t_end, k0_up=5, k0_down=k0_down)
    probes = [sh.nearest(0.0, 0.5), sh.nearest(0.5, 0.5), sh.nearest(1.0, 0.5)]
    return Problem("C1", sh, [model], np.zeros(sh.n, np.uint8), [(nodes, 0.0, 1.0, amp, None)], cfg, probes)


def c2(model="ohara2011-epi", t_end=500.0, k0_down=3, amplitude=C2_AMPLITUDE, radius=C2_RADIUS,
       scheme=api.Scheme.DAETI) -> Problem:
    sh = api.Sheet(5.0, 5.0, 0.025, math.pi / 4, d0_myocyte=0.0012, rho=0.25)
    nodes = sh.select("disc", cx=0.0, cy=0.0, radius=radius)
    cfg = api.SchemeConfig(scheme=scheme, dt_ms=0.1, t_end_ms=t_end, k0_up=5, k0_down=k0_down)
    probes = [sh.nearest(0.0, 0.0), sh.nearest(2.5, 2.5), sh.nearest(5.0, 5.0)]
    return Problem("C2", sh, [model], np.zeros(sh.n, np.uint8), [(nodes, 0.0, 1.0, amplitude, None)], cfg, probes)


# C3 stimuli by the reference's rule, 2 x diastolic_threshold (stimulus.cpp:115-157) of each stimulus on the
# C3 grid (tools/threshold_c3.py, searched on the device, window 200 ms; profiles/r02_thresholds.txt):
#   S1: left-edge strip x <= 0.05 cm: 46.0 mV/ms at h = 0.005 and at h = 0.01 -> 92 mV/ms (a single node
#       line at h = 0.005 does not propagate even at the search's 1000 mV/ms cap: too thin a source);
#   S2: quadrant [0, 2.5]^2 cm: 35.0 mV/ms (h = 0.01) -> 70 mV/ms.
C3_S1_AMPLITUDE = 92.0
C3_S1_STRIP = 0.05
C3_S2_AMPLITUDE = 70.0
# C3 tissue state: ORd-epi paced to steady state at a 600 ms cycle (20 beats, 70 mV/ms = 2 x the no-drain
# threshold, 1 ms; APD90 ~227 ms). From the rest state (APD90 ~290 ms on the first beat) or paced at 1 Hz
# (APD90 ~242 ms) the S2 at 300 ms finds the S1-activated tissue still refractory and no re-entry follows;
# at 500-600 ms cycles the S2 wave re-enters around the scar (tools/c3_reentry.py,
# profiles/r02_c3_reentry.txt).
C3_PACING = (0, 600.0, 20, 70.0, 1.0)


def c3(t_end=1000.0, k0_down=3, seed=2011, amplitude=C3_S1_AMPLITUDE, h=0.005, size=5.0,
       amplitude_s2=C3_S2_AMPLITUDE) -> Problem:
    """Pathological sheet (EXTENSION; parity pinned to the C oracle only).

    Central scar (r = 1 cm): elements with D = 0 and passive nodes; border
    zone (1-1.5 cm): D x 0.5 and per-node GKr x U(0.8, 1.2) drawn from
    std::mt19937_64(seed) in ascending node order (uniform_mt64). S1: left-
    edge strip x <= 0.05 cm at t = 0; S2: quadrant [0, size/2]^2 at t = 300
    ms (cross-field to the S1 wave); both 1 ms at 2 x their diastolic
    threshold on this grid (constants above).
    """
    nx = int(round(size / h))
    c = size / 2.0
    # element centroids
    ex = (np.arange(nx) + 0.5) * h
    X, Y = np.meshgrid(ex, ex)
    r = np.hypot(X - c, Y - c).ravel()
    scale = np.where(r <= 1.0, 0.0, np.where(r <= 1.5, 0.5, 1.0))
    sh = api.Sheet(size, size, h, 0.0, d0_myocyte=0.001, rho=1.0, elem_scale=scale)
    rn = np.hypot(sh.coords[:, 0] - c, sh.coords[:, 1] - c)
    model_of_node = np.where(rn < 1.0 - 1e-9, 1, 0).astype(np.uint8)  # strictly inside the scar: passive
    gkr = np.ones(sh.n)
    bz = (rn >= 1.0) & (rn <= 1.5)
    gkr[bz] = uniform_mt64(seed, int(bz.sum()), 0.8, 1.2)  # border-zone nodes in ascending index
    s1 = sh.select("x_le", value=C3_S1_STRIP)
    s2 = sh.select("rectangle", x0=0.0, x1=c, y0=0.0, y1=c)
    cfg = api.SchemeConfig(scheme=api.Scheme.DAETI, dt_ms=0.1, t_end_ms=t_end, k0_up=5, k0_down=k0_down)
    probes = [sh.nearest(0.5, c), sh.nearest(c, 0.5), sh.nearest(size - 0.5, c)]
    return Problem("C3", sh, ["ohara2011-epi", "passive"], model_of_node,
                   [(s1, 0.0, 1.0, amplitude, None), (s2, 300.0, 1.0, amplitude_s2, None)], cfg, probes, gkr,
                   notes="extension: scar/passive/GKr jitter (parity unpinned by the reference)", pacing=C3_PACING)


def site_centers(lx, ly, n_sites, seed):
    """Endocardial stimulus sites of config 5: 2 n_sites draws of std::mt19937_64(seed), site k at
    (lx * u[2k], ly * u[2k+1])."""
    u = uniform_mt64(seed, 2 * n_sites, 0.0, 1.0)
    return [(lx * u[2 * k], ly * u[2 * k + 1]) for k in range(n_sites)]


def slab(lx, ly, lz, h, model="ohara2011-epi", t_end=10.0, k0_down=3, amplitude=150.0, stim="face", seed=2011,
         n_sites=16, site_radius=0.1, d_long=0.0012, rho=0.25) -> Problem:
    """3D slab (EXTENSION; oracle-pinned). Fibres rotate +60 -> -60 deg from endocardium (z = 0) to
    epicardium, D_l:D_t = 4:1 (rho 0.25), D_l = 0.0012 cm^2/ms (as C2). Stimulus on z = 0: the whole
    face ("face", config 4) or n_sites seeded random discs ("sites", config 5; site_centers)."""
    sl = api.Slab3D(lx, ly, lz, h, d_long=d_long, rho=rho)
    if stim == "face":
        nodes = sl.face_z0()
    else:
        centers = site_centers(lx, ly, n_sites, seed)
        nodes = sl.discs_z0(centers, site_radius)
    cfg = api.SchemeConfig(scheme=api.Scheme.DAETI, dt_ms=0.1, t_end_ms=t_end, k0_up=5, k0_down=k0_down)
    probes = [sl.nearest(lx / 2, ly / 2, 0.0), sl.nearest(lx / 2, ly / 2, lz), sl.nearest(lx, ly, lz / 2)]
    return Problem(f"slab{sl.nx1}x{sl.ny1}x{sl.nz1}", sl, [model], np.zeros(sl.n, np.uint8),
                   [(nodes, 0.0, 1.0, amplitude, None)], cfg, probes, notes="extension: 3D slab")


def c4(t_end=500.0, **kw) -> Problem:
    """BASELINE configs[3]: 5x5x1 cm, h = 0.02 (251x251x51 = 3.2M nodes), endocardial face stimulus."""
    return slab(5.0, 5.0, 1.0, 0.02, t_end=t_end, **kw)


# C5 endocardial sites: discs of radius 0.2 cm at 450 mV/ms for 1 ms. A site's threshold (the reference's
# bisection rule applied in 3D, tools/threshold_c5_site.py: a node >= 0.5 cm away activates within 30 ms)
# lies in (360, 400] mV/ms; 2x that drives the ORd forward-Euler reaction past its stability limit under DAETI
# at dt 0.1 ms (512 mV/ms aborts at t = 0.99 ms), so the largest tested amplitude below it that propagates is
# used. Radius-0.1 cm sites do not propagate at any amplitude below the abort (profiles/r02_c5_sites.txt).
C5_SITE_RADIUS = 0.2
C5_AMPLITUDE = 450.0


def c5(t_end=5.0, **kw) -> Problem:
    """BASELINE configs[4]: 10x10x2 cm, h = 0.01 (1001x1001x201 = 201M nodes), 16 random endocardial sites."""
    kw.setdefault("amplitude", C5_AMPLITUDE)
    kw.setdefault("site_radius", C5_SITE_RADIUS)
    return slab(10.0, 10.0, 2.0, 0.01, t_end=t_end, stim="sites", **kw)


def c5_subslab(ly=0.2, t_end=5.0, n_sites=16, **kw) -> Problem:
    """A full-cross-section y-sub-slab of config 5 for parity at BASELINE resolution: 10 x ly x 2 cm at
    h = 0.01 (1001 x (ly/h + 1) x 201 nodes; ly = 0.2 -> 4.2M nodes), same fibres, conductivities and
    stimulus kind (n_sites seeded endocardial discs over its own face)."""
    kw.setdefault("amplitude", C5_AMPLITUDE)
    kw.setdefault("site_radius", C5_SITE_RADIUS)
    return slab(10.0, ly, 2.0, 0.01, t_end=t_end, stim="sites", n_sites=n_sites, **kw)
