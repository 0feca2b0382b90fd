"""Diagnostic: per-step reaction time vs the step's k distribution on C2 (one B200)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import _lib as L, problems  # noqa: E402

p = problems.c2()
integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=p.model_of_node)
integ.upload(p.initial_state())
integ.run_begin()
integ.run_steps(0, 1)
integ.run_sync()
lib = L.lib()
n = integ.info.n_steps
kh_prev = integ.k_histogram()
rows = []
for s in range(1, n - 1):
    st, re, di = np.zeros(1), np.zeros(1), np.zeros(1)
    assert lib.cwg_bench_steps(integ._h, s, 1, 0, 0, L.dp(st), L.dp(re), L.dp(di)) == 0
    kh = integ.k_histogram()
    d = kh - kh_prev
    kh_prev = kh
    kmax = int(np.nonzero(d)[0].max())
    rows.append((s, re[0], di[0], kmax, int((d * np.arange(len(d))).sum()), int(d[kmax])))
a = np.array(rows)
np.save("gpurun_out/c2_steps.npy", a)
for lo, hi in [(1, 500), (500, 1500), (1500, 3000), (3000, 4999)]:
    sel = (a[:, 0] >= lo) & (a[:, 0] < hi)
    print(f"steps {lo}-{hi}: react mean {a[sel,1].mean()*1e3:.1f} us  p90 {np.percentile(a[sel,1],90)*1e3:.1f}  "
          f"kmax mean {a[sel,3].mean():.1f}  evals mean {a[sel,4].mean():.0f}  n_at_kmax {a[sel,5].mean():.0f}")
for k in range(3, 11):
    sel = a[:, 3] == k
    if sel.any():
        print(f"kmax={k}: {sel.sum()} steps, react mean {a[sel,1].mean()*1e3:.1f} us")
