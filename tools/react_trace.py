"""Diagnostic: where one step's device time goes (CWG_REACT_TRACE=1 python tools/react_trace.py [cN] [step ...]).

Runs the C2 problem to `step`, then times that step the way bench.py does
(256 MiB L2 flush, then the step graph between CUDA events) while the
reaction kernel stamps %globaltimer per block. Prints the event-timed
reaction phase next to the kernel's own span (first block start -> last
block done): the difference is launch + completion latency around the
kernel, which no kernel change can remove.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04747_b200 as cw  # noqa: E402
from paper_2011_04747_b200 import _lib as L, problems  # noqa: E402

assert os.environ.get("CWG_REACT_TRACE"), "set CWG_REACT_TRACE=1"
lib = L.lib()
args = sys.argv[1:]
cfg = args.pop(0) if args and args[0].startswith("c") else "c2"
p = getattr(problems, cfg)()
integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=p.model_of_node)
integ.upload(p.initial_state())
integ.run_begin()
pos = 0
for step in sorted(int(a) for a in args) or [2000, 4000]:
    integ.run_steps(pos, step - pos)  # bring the wave to this step
    integ.run_sync()
    pos = step + 1
    st, re, di = np.zeros(1), np.zeros(1), np.zeros(1)
    flush = int(os.environ.get("FLUSH_MB", "256")) << 20
    assert lib.cwg_bench_steps(integ._h, step, 1, flush, 0, L.dp(st), L.dp(re), L.dp(di)) == 0
    buf = np.zeros(16 * 4096, np.uint64)
    assert lib.cwg_react_trace(buf.ctypes.data, len(buf)) == 0
    t = buf.reshape(4096, 16).astype(np.int64)
    t = t[t[:, 15] > 0]
    t0 = t[:, 15].min()
    done = (t[:, 0] - t0) / 1e3
    print(f"{cfg} step {step}: reaction phase {re[0] * 1e3:.1f} us event-timed; kernel span {done.max():.1f} us "
          f"({len(t)} blocks start within {(t[:, 15].max() - t0) / 1e3:.2f} us; block done: min {done.min():.1f}, "
          f"median {np.median(done):.1f}, max {done.max():.1f} us); diffusion + recording {di[0] * 1e3:.1f} us")
    late = np.sort(done[done > np.median(done) + 3.0])
    if len(late):
        print(f"  {len(late)} blocks finish > 3 us after the median (a second lane round): "
              f"done at {', '.join(f'{x:.1f}' for x in np.percentile(late, [0, 25, 50, 75, 100]))} us (0/25/50/75/100%)")
integ.close()
