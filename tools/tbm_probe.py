import sys, os, math
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import api, problems
sh = cw.Sheet(8.0, 4.0, 0.01, math.pi / 4, d0_myocyte=0.0017, rho=0.25)
nodes = sh.select("x_le", value=0.05)
p = problems.Problem("tb", sh, ["aliev-panfilov"], np.zeros(sh.n, np.uint8), [(nodes, 0.0, 1.0, 100.0, None)],
                     api.SchemeConfig(dt_ms=0.3, t_end_ms=0.9), [0])
r = cw.run_simulation(p.initial_state(), p.setup(), p.cfg)
print("ok", r.final_state.v[:3])
