"""Host vs device assembly of BASELINE configs[2] (C3, 1001 x 1001 with the scar / border-zone D scale):
wall time of the host restatement (std::sort triplet assembly, = the reference's algorithm), of the
device path (mesh on the host + cwg_sheet2d_assemble), and how many diagonal entries differ (ulp)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import ctypes as C
import numpy as np
import paper_2011_04747_b200 as cw
from paper_2011_04747_b200 import _lib as L

h, size = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005, 5.0
nx = int(round(size / h))
ex = (np.arange(nx) + 0.5) * h
X, Y = np.meshgrid(ex, ex)
r = np.hypot(X - size / 2, Y - size / 2).ravel()
scale = np.where(r <= 1.0, 0.0, np.where(r <= 1.5, 0.5, 1.0))
cw.Sheet(1.0, 1.0, 0.05, 0.0, d0_myocyte=0.001, rho=1.0, elem_scale=np.ones(400), assembly="device")  # warm-up
t0 = time.perf_counter()
host = cw.Sheet(size, size, h, 0.0, d0_myocyte=0.001, rho=1.0, elem_scale=scale)
t1 = time.perf_counter()
dev = cw.Sheet(size, size, h, 0.0, d0_myocyte=0.001, rho=1.0, elem_scale=scale, assembly="device")
t2 = time.perf_counter()
dts = C.c_double()
err = L.cwg_error()
t3 = time.perf_counter()
L.lib().cwg_sheet2d_assemble(C.byref(dev.op.desc), 0, None, None, None, None, C.byref(dts), C.byref(err))
t4 = time.perf_counter()
csr = dev.op.csr()
rows = np.repeat(np.arange(host.n), np.diff(host.op.row_ptr))
diag = host.op.col == rows
u = np.abs(csr.val.view(np.int64) - host.op.val.view(np.int64))
print(f"C3 grid {nx + 1}^2 = {host.n} nodes, nnz {len(host.op.val)}")
print(f"host assembly (cwg_sheet_build, std::sort triplets): {1e3 * (t1 - t0):.1f} ms")
print(f"device path (host mesh + device assembly + dt_s): {1e3 * (t2 - t1):.1f} ms; "
      f"cwg_sheet2d_assemble alone (dt_s only): {1e3 * (t4 - t3):.1f} ms")
print(f"mass bitwise equal: {np.array_equal(csr.lumped_mass.view(np.int64), host.op.lumped_mass.view(np.int64))}; "
      f"off-diagonals bitwise equal: {np.array_equal(csr.val[~diag].view(np.int64), host.op.val[~diag].view(np.int64))}; "
      f"diagonals differing: {int((u[diag] > 0).sum())} of {int(diag.sum())} (max {int(u[diag].max())} ulp); "
      f"dt_s host {host.op.dt_s!r} device {dev.op.dt_s!r}")
