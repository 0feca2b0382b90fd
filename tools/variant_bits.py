"""Do the ORd launch-shape variants give the same bits? C4 for a few ms with CWG_ORD_VARIANT forced per integrator;
prints max |dV| and the number of differing V / state entries against variant 1 (the throughput shape)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems
p = problems.c4(t_end=float(sys.argv[1]) if len(sys.argv) > 1 else 3.0)
setup = p.setup()
res = {}
for v in sys.argv[2].split() if len(sys.argv) > 2 else ("1", "0"):
    os.environ["CWG_ORD_VARIANT"] = v
    r = cw.run_simulation(p.initial_state(), setup, p.cfg)
    res[v] = r.final_state
    b = res["1"]
    dv = np.abs(r.final_state.v - b.v)
    print(f"variant {v}: V differs at {int((r.final_state.v != b.v).sum())} nodes (max {dv.max():.3e} mV), "
          f"states differ at {int((r.final_state.s != b.s).sum())} entries", flush=True)
