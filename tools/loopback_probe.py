"""Loopback (CWG_LOOPBACK=1) run of C4 split into y-slab contexts on one device: usage loopback_probe.py <t_end_ms> <world>; prints the cwg_loopback_steps status."""
import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
os.environ["CWG_LOOPBACK"] = "1"
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import problems, _lib as L
p = problems.c4(t_end=float(sys.argv[1]))
world = int(sys.argv[2])
setup = p.setup()
integs = [cw.StrangIntegrator(setup, p.cfg, model_of_node=p.model_of_node, rank=r, world=world) for r in range(world)]
hs = (C.c_void_p * world)(*[it._h.value for it in integs])
st = p.initial_state()
for it in integs:
    it.upload(st); it.run_begin()
rc = L.lib().cwg_loopback_steps(hs, world, 0, integs[0].info.n_steps)
print("rc", rc, L.lib().cwg_last_error().decode())
