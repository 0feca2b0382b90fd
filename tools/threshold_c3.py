"""Stimulus amplitudes of BASELINE configs[2] (C3) by the reference's own rule: 2 x diastolic_threshold
(stimulus.cpp:115-157) of each stimulus on the C3 grid (5 x 5 cm, h = 0.005, D = 0.001 isotropic, ORd-epi),
searched on the device (cwg_diastolic_threshold). The scar is left out of the search sheet: its
conductivity is zero and the search probe is the node farthest from the stimulus, which a scar would
disconnect; the threshold is set by the source-sink balance at the stimulus, centimetres from the scar.
window_ms = 200 (the default 50 ms cannot reach a probe 3.5-5 cm away at ~0.05 cm/ms).
  S1: left-edge strip x <= 0.05 cm (a single node line at h = 0.005 does not propagate even at the search's
      1000 mV/ms upper bracket: its source is too thin for the sink, cwg run 2026-10-20);
  S2: quadrant [0, 2.5]^2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402

h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005
sh = cw.Sheet(5.0, 5.0, h, 0.0, d0_myocyte=0.001, rho=1.0)
opts = cw.ThresholdOptions(window_ms=200.0)
which = sys.argv[2:] or ["S1", "S2"]
cases = {"S1": ("S1 strip x<=0.05", lambda: sh.select("x_le", value=0.05)),
         "S2": ("S2 quadrant [0,2.5]^2", lambda: sh.select("rectangle", x0=0.0, x1=2.5, y0=0.0, y1=2.5))}
for name, nodes in ((cases[k][0], cases[k][1]()) for k in which):
    t0 = time.perf_counter()
    thr, probe = cw.diastolic_threshold(sh, cw.make_model("ohara2011-epi"), nodes, opts, return_probe=True)
    print(f"h={h} {name}: threshold {thr} mV/ms (2x = {2 * thr}), probe node {probe}, "
          f"{time.perf_counter() - t0:.1f} s", flush=True)
