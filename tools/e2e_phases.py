"""Phase timing of the end-to-end path on C4 (create / upload / steps / download / maps), with cwg_create's own phases (CWG_TRACE_CREATE)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["CWG_TRACE_CREATE"] = "1"
import numpy as np, torch
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems
p = problems.c4(t_end=2.5)
setup = p.setup()
st = p.initial_state()
pin = lambda a: (lambda t: (t.copy_(torch.from_numpy(a)), t.numpy())[1])(torch.empty(a.shape, dtype=torch.float64, pin_memory=True))
if os.environ.get("PINNED", "1") == "1":  # as bench.py's e2e: host state in pinned memory
    st.v, st.s, st.last_dvdt = pin(st.v), pin(st.s), pin(st.last_dvdt)
fin = st.copy()
fin.v, fin.s, fin.last_dvdt = pin(fin.v), pin(fin.s), pin(fin.last_dvdt)
pinned = lambda dt: torch.empty(p.n, dtype=dt, pin_memory=True).numpy()
maps_out = tuple(cw.ScalarMap(pinned(torch.float64), pinned(torch.bool)) for _ in range(2))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    integ = cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node)
    t1 = time.perf_counter()
    integ.upload(st); t2 = time.perf_counter()
    integ.run_begin(); t3 = time.perf_counter()
    integ.run_steps(0, integ.info.n_steps); integ.run_sync(); t4 = time.perf_counter()
    t5 = time.perf_counter()
    integ.download(fin); t6 = time.perf_counter()
    integ.traces(); integ.maps(maps_out); t7 = time.perf_counter()
    integ.close(); t8 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} upload {1e3*(t2-t1):.1f} begin {1e3*(t3-t2):.1f} steps {1e3*(t4-t3):.1f} "
          f"download {1e3*(t6-t5):.1f} maps {1e3*(t7-t6):.1f} close {1e3*(t8-t7):.1f} ms", flush=True)
