"""Batched single-cell pacing: an ORd-epi cycle-length sweep on the GPU
(cwg_pace_cells, one thread per cell) vs the reference's pace_to_steady_state
per cell on this host (oracle/_ref, one cell timed, scaled by cells / threads)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2011_04747_b200 as cw  # noqa: E402

n, beats = int(os.environ.get("PACE_N", "4736")), int(os.environ.get("PACE_BEATS", "3"))
cls = np.linspace(300.0, 1000.0, n)
cw.pace_cells("ohara2011-epi", cls[:8], 1, 80.0, 1.0)  # warm-up
t0 = time.perf_counter()
res, errs = cw.pace_cells("ohara2011-epi", cls, beats, 80.0, 1.0)
t_gpu = time.perf_counter() - t0
print(f"gpu: {n} cells x {beats} beats (CL 300-1000 ms) in {t_gpu:.2f} s; failures {sum(e is not None for e in errs)}")
try:
    import refpy
    if refpy.available():
        t0 = time.perf_counter()
        refpy.pace("ohara2011-epi", float(cls[n // 2]), beats, 80.0, 1.0)
        t1 = time.perf_counter() - t0
        th = os.cpu_count()
        print(f"reference: one cell ({cls[n // 2]:.0f} ms CL) {t1:.2f} s -> {n} cells on {th} threads ~{t1 * n / th:.0f} s")
except Exception as e:  # noqa: BLE001
    print("reference timing skipped:", e)
