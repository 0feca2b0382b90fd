"""The C++ drop-in (include/cardwave_gpu.hpp) side by side with the unmodified
reference in one process: oracle/_ref/shim_parity runs cardwave::run_simulation
and cardwave::gpu::run_simulation on the same reference-built problem."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_parity")


@pytest.mark.parametrize("mode", ["diffusion", "ap", "ord", "abort", "c1", "c2", "advance", "resident"])
def test_cpp_dropin_matches_reference(mode):
    if not os.path.exists(EXE):
        pytest.skip("shim_parity not built (needs /root/reference at build time)")
    # c1 / c2: BASELINE configs[0] / configs[1] over their whole 400 / 500 ms runs (ORd-epi, the reference
    # on all host threads: ~5 s / ~25 s), max|dV| <= 1e-6 mV, identical k-histograms, LAT validity, snapshots
    args = [EXE, mode]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    if mode == "abort":
        assert line["ref_abort"][0] == 16 and line["match"]
        assert line["snapshots"][0] == line["snapshots"][1] == 5  # t = 0, 0.5, ..., 2.0
    elif mode in ("ap", "ord", "c1", "c2"):
        assert line["snapshots"][0] == line["snapshots"][1] > 1 and line["pass"]
    elif mode in ("advance", "resident"):
        assert line["steps"] == 200 and line["pass"]
