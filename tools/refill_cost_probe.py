"""What does a node's write-back + refill cost the ORd reaction, against one rates evaluation? Runs the first steps
of C4 without its stimulus (tissue at rest, so every node has k = k0) with k0_up = k0_down = K for several
K: ms per step = N (K E + R) separates the per-evaluation cost E from the per-node cost R. Whole
steps are timed (diffusion is ~4% of a C4 step and the same in every run)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems, api, _lib as L
import torch

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rows = []
for tag, scheme, k0 in (("k3", api.Scheme.DAETI, 3), ("k4", api.Scheme.DAETI, 4), ("k6", api.Scheme.DAETI, 6),
                        ("k9", api.Scheme.DAETI, 9), ("k12", api.Scheme.DAETI, 12)):
    p = problems.c4(t_end=(steps + 4) * 0.1)
    p.stimuli = []  # tissue at rest: every node has k = k0 exactly
    p.cfg = api.SchemeConfig(scheme=scheme, dt_ms=0.1, t_end_ms=(steps + 4) * 0.1, k0_up=k0, k0_down=k0)
    setup = p.setup()
    integ = cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node)
    integ.upload(p.initial_state())
    integ.run_begin()
    integ.run_steps(0, 4)
    integ.run_sync()
    ev0 = int(L.lib().cwg_reaction_evals(integ._h))
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    integ.run_steps(4, steps)
    integ.run_sync()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    ev = (int(L.lib().cwg_reaction_evals(integ._h)) - ev0) / steps
    rows.append((tag, ms, ev / p.n))
    print(json.dumps({"run": tag, "ms_per_step": ms, "mean_k": ev / p.n, "ns_per_eval": ms * 1e6 / ev}))
    integ.close()
# least squares ms = N (k E + R)
A = np.array([[r[2], 1.0] for r in rows]); y = np.array([r[1] for r in rows])
(E, R), *_ = np.linalg.lstsq(A, y, rcond=None)
print("fit: per-evaluation %.4f ms per N nodes, per-node (refill + diffusion share) %.4f ms; R / E = %.2f" % (E, R, R / E))
