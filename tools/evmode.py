"""Diagnostic: C2 per-step device time under three event placements (cwg_bench_steps split_phases 0/1/2)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import _lib as L, problems  # noqa: E402

p = problems.c2()
lib = L.lib()
for mode in (0, 2, 1, 0, 2):
    integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=p.model_of_node)
    integ.upload(p.initial_state())
    integ.run_begin()
    integ.run_steps(0, 10)
    integ.run_sync()
    K = 2000
    st, re, di = np.zeros(K), np.zeros(K), np.zeros(K)
    assert lib.cwg_bench_steps(integ._h, 10, K, 256 << 20, mode, L.dp(st), L.dp(re), L.dp(di)) == 0
    print(f"mode {mode}: step {st.mean()*1e3:.2f} us (first phase {re.mean()*1e3:.2f}, second {di.mean()*1e3:.2f})")
    integ.close()
