"""diastolic_threshold for ORd-epi on the C1 sheet (x <= 0 line), the case the
survey timed in the reference (808 s on 4 threads, threshold 296 mV/ms).
Optionally also runs the reference itself (oracle/_ref) on this host: --ref."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2011_04747_b200 as cw  # noqa: E402

sh = cw.Sheet(1.0, 1.0, 0.01, 0.0, d0_myocyte=0.001, rho=1.0)
nodes = sh.select("x_le", value=0.0)
t0 = time.perf_counter()
thr = cw.diastolic_threshold(sh, cw.make_model("ohara2011-epi"), nodes)
print(f"gpu threshold {thr} mV/ms in {time.perf_counter() - t0:.2f} s", flush=True)
if "--ref" in sys.argv:
    import refpy
    r = refpy.Sheet(1.0, 1.0, 0.01, 0.0, d0=0.001, rho=1.0)
    t0 = time.perf_counter()
    rt = r.threshold("ohara2011-epi", r.select("x_le", value=0.0))
    print(f"reference threshold {rt} mV/ms in {time.perf_counter() - t0:.1f} s ({os.cpu_count()} host threads)")
