"""Does the config-5 stimulus excite? Runs the C5 y-sub-slab (problems.c5_subslab: 10 x 0.2 x 2 cm, h = 0.01,
16 seeded endocardial discs of radius 0.1 cm) for 5 ms on the device at several amplitudes and prints how
many nodes activated (LAT at 0 mV) and the run's k-histogram."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import problems  # noqa: E402

for amp in [float(a) for a in (sys.argv[1:] or ["150", "300", "600"])]:
    for radius in (0.1, 0.2):
        p = problems.slab(10.0, 0.2, 2.0, 0.01, t_end=5.0, stim="sites", n_sites=16, amplitude=amp, site_radius=radius)
        try:
            r = cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
            print(f"amp {amp} r {radius}: stim nodes {len(p.stimuli[0][0])}, activated {int(r.lat_map.valid.sum())}, "
                  f"V max {r.final_state.v.max():.2f}, khist {r.k_histogram.tolist()}", flush=True)
        except cw.InstabilityError as e:
            print(f"amp {amp} r {radius}: InstabilityError {e}", flush=True)
