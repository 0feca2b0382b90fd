"""Does BASELINE configs[2] (C3) do what it exists for? Runs the full pathological sheet (1001 x 1001 nodes,
scar + border zone + GKr jitter, S1 at t = 0, S2 quadrant at 300 ms) for T ms on the device with a 7 x 7 grid
of probe nodes, and reports each probe's activation times (upward 0 mV crossings of its trace, record
interval 1 ms). Re-entry = activations after the S2 wave has passed (t > 300 ms + the time S2 needs to
cross the sheet), i.e. tissue re-excited with no stimulus on.
  python tools/c3_reentry.py [T_ms] [out.npz]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import problems  # noqa: E402

t_end = float(sys.argv[1]) if len(sys.argv) > 1 else 1000.0
out = sys.argv[2] if len(sys.argv) > 2 else None
p = problems.c3(t_end=t_end)
xs = np.linspace(0.25, 4.75, 7)
p.probes = [p.sheet.nearest(x, y) for y in xs for x in xs]
st = p.initial_state()
paced = os.environ.get("PACED")  # "CL,beats": start ORd-epi nodes from pace_to_steady_state (ionic.cpp:122-167)
if paced:
    cl, beats = paced.split(",")
    pr = cw.pace_to_steady_state("ohara2011-epi", float(cl), int(beats), 80.0, 1.0)
    print(f"paced ORd-epi at CL {cl} ms x {beats}: APD90 of the last beats {pr.apd90_ms[-3:]}, "
          f"max rel change {pr.max_rel_change:.2e}", flush=True)
    st = cw.make_initial_state(p.n, [cw.make_model(m) for m in p.models], p.model_of_node,
                               initial_per_model=[pr.state, None])
t0 = time.perf_counter()
r = cw.run_simulation(st, p.setup(), p.cfg)
wall = time.perf_counter() - t0
lat = r.lat_map
print(f"C3 {t_end} ms: {wall:.1f} s wall, activated {int(lat.valid.sum())} of {p.n} nodes "
      f"(passive scar nodes {int((p.model_of_node == 1).sum())}), k-hist {r.k_histogram.tolist()}", flush=True)
acts = []
for q, tr in enumerate(r.traces):
    v = tr.v_mv
    up = np.flatnonzero((v[:-1] < 0.0) & (v[1:] >= 0.0))
    times = tr.t_ms[up + 1]
    acts.append(times)
    x, y = p.sheet.coords[p.probes[q]]
    print(f"probe ({x:.2f}, {y:.2f}) mid={int(p.model_of_node[p.probes[q]])}: activations at "
          f"{', '.join(f'{t:.0f}' for t in times)} ms", flush=True)
late = [t for a in acts for t in a if t > 450.0]
print(f"activations after 450 ms (no stimulus on): {len(late)} across "
      f"{sum(1 for a in acts if np.any(a > 450.0))} probes -> re-entry {'YES' if late else 'NO'}", flush=True)
if out:
    np.savez_compressed(out, t=r.traces[0].t_ms, v=np.array([tr.v_mv for tr in r.traces]),
                        probes=np.array(p.probes), xy=p.sheet.coords[p.probes], lat=lat.value.reshape(1001, 1001)[::5, ::5],
                        lat_valid=lat.valid.reshape(1001, 1001)[::5, ::5])
