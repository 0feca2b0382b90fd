"""How much does C3's list bin (ORd nodes outside the passive scar) cost the reaction? Runs C3 for N steps as
configured (two bins: ORd list + passive list) and with every node ORd (one dense bin; the scar's D = 0 keeps its
nodes isolated), and prints reaction evaluations per second of each (bench-style step graph, L2 flushed)."""
import os, sys, json, subprocess
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems, _lib as L
import ctypes as C
import torch

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for dense in (False, True):
    p = problems.c3(t_end=(steps + 20) * 0.1)
    if dense:
        p.model_of_node = np.zeros(p.n, np.uint8)
        p.models = ["ohara2011-epi"]
        p.pacing = None
    setup = p.setup()
    integ = cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node)
    integ.upload(p.initial_state())
    integ.run_begin()
    integ.run_steps(0, 20)
    integ.run_sync()
    ev0 = int(L.lib().cwg_reaction_evals(integ._h))
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    integ.run_steps(20, steps)
    integ.run_sync()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    ev = int(L.lib().cwg_reaction_evals(integ._h)) - ev0
    print(json.dumps({"dense": dense, "ms_per_step": ms / steps, "evals_per_step": ev / steps, "evals_per_s": ev / (ms / 1e3)}))
    integ.close()
