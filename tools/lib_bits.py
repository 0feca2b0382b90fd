"""Bitwise comparison of two library builds on one problem: run it with CWG_LIB_PATH=<lib> and save the final
state (python tools/lib_bits.py run <out.npz> [c4|c2|c3] [t_end]; keep the files outside gpurun_out/: a C4 state is 1 GB),
then compare two saved runs
(python tools/lib_bits.py cmp a.npz b.npz)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        d = a[k] != b[k]
        print(k, "differ at", int(d.sum()), "of", d.size, "max |diff|", float(np.max(np.abs(a[k] - b[k]))) if d.any() else 0.0)
    raise SystemExit
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems
cfg = sys.argv[3] if len(sys.argv) > 3 else "c4"
t_end = float(sys.argv[4]) if len(sys.argv) > 4 else 8.0
p = getattr(problems, cfg)(t_end=t_end)
r = cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
np.savez(sys.argv[2], v=r.final_state.v, s=r.final_state.s, kh=r.k_histogram, lat=np.nan_to_num(r.lat_map.value))
