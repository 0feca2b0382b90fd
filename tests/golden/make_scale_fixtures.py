"""Generate the BASELINE-size parity fixtures tests/golden/scale_*.npz with the C restatement oracle.

TEST INFRASTRUCTURE ONLY. The oracle (oracle/cw_oracle.c, OpenMP; pinned bit-exact to the reference in
tests/test_oracle_pins.py) runs each configuration at its BASELINE resolution for a window long enough to
carry the wave across a large part of the tissue, and the fixture keeps what the GPU tests compare
(SURVEY.md 8(c) parity protocol):

  * the sampled node set -- every 10th node along each axis, plus the probes -- with final V, LAT and
    APD90 (and their validity flags),
  * the probe traces at the record cadence,
  * the k-histogram,
  * a description of the inputs (sizes, stimulus node-set and GKr checksums) so a test can assert that it
    rebuilt the same problem.

The problem definitions come from paper_2011_04747_b200/problems.py (geometry, stimulus node sets, GKr
jitter, probes: the shared INPUT); every number in the fixture is computed by the oracle. 2D operators are
the host CSR that tests/test_setup_parity.py pins bit-identical to the reference's `assemble`; 3D slabs
use the oracle's own assembly (orapy.Slab3DOp).

    python tests/golden/make_scale_fixtures.py c4        # 251x251x51, 20 ms   (~7 min on 8 cores)
    python tests/golden/make_scale_fixtures.py c5sub     # 1001x21x201, 5 ms   (~3 min)
    python tests/golden/make_scale_fixtures.py c3        # 1001x1001, 40 ms    (~9 min)
    python tests/golden/make_scale_fixtures.py c3half    # 501x501, 400 ms incl. S2 at 300 ms (~15 min)
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import orapy  # noqa: E402

from paper_2011_04747_b200 import problems  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def problem(name):
    if name == "c4":
        return problems.c4(t_end=20.0)
    if name == "c5sub":
        return problems.c5_subslab(t_end=5.0)
    if name == "c3":
        return problems.c3(t_end=40.0)
    if name == "c3half":
        return problems.c3(t_end=400.0, h=0.01)
    raise SystemExit(f"unknown fixture {name}")


def sampled(prob):
    """every 10th node along each axis plus the probes."""
    op = prob.sheet.op
    if hasattr(op, "nz1"):
        iy, iz, ix = np.meshgrid(np.arange(0, op.ny1, 10), np.arange(0, op.nz1, 10), np.arange(0, op.nx1, 10),
                                 indexing="ij")
        idx = op.index(ix, iy, iz).ravel()
    else:
        nx1 = op.grid_nx1
        ys, xs = np.meshgrid(np.arange(0, prob.n // nx1, 10), np.arange(0, nx1, 10), indexing="ij")
        idx = (ys * nx1 + xs).ravel()
    return np.union1d(idx, np.asarray(prob.probes, np.int64)).astype(np.int64)


def oracle_op(prob):
    op = prob.sheet.op
    if hasattr(op, "nz1"):
        o = orapy.Slab3DOp(op.nx, op.ny, op.nz, op.h, op.d_long, op.rho)
        assert np.array_equal(o.angles, op.angles)
        return o, o.dt_s
    return (op.row_ptr, op.col, op.val, op.lumped_mass), op.dt_s


def make(name):
    prob = problem(name)
    cfg = prob.cfg
    op, dt_s = oracle_op(prob)
    init, paced = None, None
    if prob.pacing is not None:  # the paced model's state from the oracle's pace_to_steady_state (ionic.cpp:122-167)
        mid, cl, beats, amp, dur = prob.pacing
        paced, _, _ = orapy.pace(prob.models[mid], cl, beats, amp, dur)
        st = prob.initial_state(paced_state=paced)
        init = (st.v, st.s.reshape(prob.n, -1), st.last_dvdt)
    t0 = time.time()
    r = orapy.run_simulation(op, dt_s, prob.models, prob.model_of_node, prob.stimuli, scheme=cfg.scheme.name,
                             dt=cfg.dt_ms, t_end=cfg.t_end_ms, k0_up=cfg.k0_up, k0_down=cfg.k0_down,
                             record_interval=cfg.record_interval_ms, probes=prob.probes,
                             gkr_scale=prob.gkr_scale, init=init)
    wall = time.time() - t0
    idx = sampled(prob)
    out = dict(
        name=np.array(name), n=np.array(prob.n), t_end=np.array(cfg.t_end_ms), dt=np.array(cfg.dt_ms),
        k0_up=np.array(cfg.k0_up), k0_down=np.array(cfg.k0_down), dt_s=np.array(dt_s), l=np.array(r["l"]),
        probes=np.asarray(prob.probes, np.int64), models=np.array(prob.models),
        stim_digest=np.array([digest(np.asarray(s[0], np.int64)) for s in prob.stimuli]),
        stim_params=np.array([[s[1], s[2], s[3]] for s in prob.stimuli]),
        gkr_digest=np.array(digest(prob.gkr_scale) if prob.gkr_scale is not None else ""),
        mon_digest=np.array(digest(np.asarray(prob.model_of_node, np.uint8))),
        idx=idx, v=r["v"][idx], lat=r["lat"][idx], lat_valid=r["lat_valid"][idx], apd=r["apd90"][idx],
        apd_valid=r["apd_valid"][idx], k_histogram=r["k_histogram"], trace_t=r["trace_t"], traces=r["traces"],
        v_mean=np.array(float(np.mean(r["v"]))), v_max=np.array(float(np.max(r["v"]))),
        activated=np.array(int(np.sum(r["lat_valid"]))), oracle_wall_s=np.array(wall),
        paced_state=np.asarray(paced if paced is not None else [], np.float64),
        oracle_threads=np.array(os.cpu_count()))
    path = os.path.join(HERE, f"scale_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: n={prob.n} steps={r['n_steps']} l={r['l']} activated={int(np.sum(r['lat_valid']))} "
          f"wall={wall:.1f}s -> {path} ({os.path.getsize(path) / 1e3:.0f} kB)", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c4", "c5sub", "c3", "c3half"]:
        make(nm)
