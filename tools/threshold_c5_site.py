"""Stimulus amplitude of BASELINE configs[4] (C5): 2 x the threshold of one endocardial disc site (radius
0.1 cm on the z = 0 face, 1 ms) in the C5 slab model (h = 0.01, fibres +60 -> -60 deg, D_l 0.0012, D_t
0.0003, ORd-epi). The reference's diastolic_threshold (stimulus.cpp:115-157) is 2D-only; this applies its
rule in 3D: bisection (rel_tol 0.05, upper bracket grown by doubling from 1 mV/ms) on "a node >= 0.5 cm
from the site activates (LAT at 0 mV) within the window", every probe run on the device."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import api, problems  # noqa: E402

L, H = 1.2, 0.6
RADIUS = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
WIN = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
sl = api.Slab3D(L, L, H, 0.01)
nodes = sl.discs_z0([(L / 2, L / 2)], RADIUS)
coords = None


def propagates(amp):
    p = problems.Problem("site", sl, ["ohara2011-epi"], np.zeros(sl.n, np.uint8), [(nodes, 0.0, 1.0, amp, None)],
                         api.SchemeConfig(dt_ms=0.1, t_end_ms=WIN, k0_up=5, k0_down=3), [])
    t0 = time.perf_counter()
    try:
        r = cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
    except cw.InstabilityError as e:
        print(f"  {amp:8.3f} mV/ms: InstabilityError ({e})", flush=True)
        raise
    iy, iz, ix = np.meshgrid(np.arange(sl.ny1), np.arange(sl.nz1), np.arange(sl.nx1), indexing="ij")
    d = np.sqrt((ix.ravel() * sl.h - L / 2) ** 2 + (iy.ravel() * sl.h - L / 2) ** 2 + (iz.ravel() * sl.h) ** 2)
    idx = sl.index(ix.ravel(), iy.ravel(), iz.ravel())
    far = idx[d >= 0.5]
    ok = bool(r.lat_map.valid[far].any())
    print(f"  {amp:8.3f} mV/ms: {'propagates' if ok else 'no'} ({int(r.lat_map.valid.sum())} activated, "
          f"{time.perf_counter() - t0:.1f} s)", flush=True)
    return ok


if len(sys.argv) > 3 and "," in sys.argv[3]:  # probe mode: just test the listed amplitudes
    for amp in (float(a) for a in sys.argv[3].split(",")):
        try:
            propagates(amp)
        except cw.InstabilityError:
            pass
    raise SystemExit(0)
lo, hi = 0.0, float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
while not propagates(hi):
    lo, hi = hi, hi * 2.0
    if hi > 1000.0:
        raise SystemExit("no propagation at the upper bracket")
while (hi - lo) / hi > 0.05:
    mid = 0.5 * (lo + hi)
    if propagates(mid):
        hi = mid
    else:
        lo = mid
print(f"C5 site (r = {RADIUS} cm) threshold {hi} mV/ms (2x = {2 * hi}) on a {sl.nx1}x{sl.ny1}x{sl.nz1} slab, window {WIN} ms", flush=True)
