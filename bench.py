#!/usr/bin/env python
"""Benchmark of the DAETI hot path on B200 (one JSON line on rank 0).

Workload (default, N = 1): BASELINE.json configs[3] ("C4"), the largest
configuration that fits one GPU: 3D ventricular slab 5 x 5 x 1 cm, h = 0.02
cm (251 x 251 x 51 = 3,213,051 nodes), fibres rotating +60 -> -60 deg from
endocardium to epicardium, D_l 0.0012 / D_t 0.0003 cm^2/ms, ORd-epi from
rest, endocardial-face stimulus (z = 0, 150 mV/ms for 1 ms), DAETI dt 0.1 ms
(k0_up 5, k0_down 3; the paper's k0_down = 1 aborts in the reference for
ORd), fp64. A "step" is one outer Strang step (the adaptive
reaction pass + 2l diffusion sub-steps + the record cadence). Default run:
the whole 500 ms simulation (W warm-up steps, then K = 5000 - W timed).
N > 1 (torchrun): strong scaling of the same C4 grid -- rank r owns a
contiguous y-slab, halo exchange of the fused diffusion launches over NCCL
(--scaling weak stacks one C4 per rank instead; --config c5 likewise splits the
201M-node slab). --config c1/c2/c3/c5 pick
the other BASELINE configurations.

metric: node-updates/s = (reaction rates evaluations + diffusion node
sub-steps) per second, whole job. Timing: CUDA events per step on the
solver's stream, with a 256 MiB L2-evicting write before every timed step
(untimed); max over ranks.

--impl reference: the reference's own CPU path on this host's physical
cores (OMP_PROC_BIND=close). C1/C2: the UNMODIFIED reference library
(oracle/_ref/libcwref.so, cardwave::StrangIntegrator::advance). C3-C5 are not
expressible in the reference (3D, scar, jitter -- SURVEY.md s0), so they run
the C restatement oracle (oracle/cw_oracle.c, pinned bit-exact to the
reference on C1/C2), kind "port". This arm never imports the product package.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "node-updates/sec (reaction+diffusion) and simulated ms per wall-s, % roofline"
UNIT = "node-updates/s"
FLUSH_BYTES = 256 << 20  # > 126 MB L2
# Executed FP64 flops per ORd rates evaluation of react_kernel<ModelOrd<epi>>
# (2*DFMA + DMUL + DADD predicated-on lane ops / evaluations), counted by ncu
# over every reaction launch of a 40-step C4 run (tools/flops_per_eval.py c4 40;
# profiles/r02g_flops_per_eval_c4.txt): 704.1 DFMA + 333.3 DMUL + 205.4 DADD
# on the final build (C2: 1,947.6; 2,152.9 before the fast path's algebraic cuts,
# 2,735.9 at the start of round 2's second session,
# profiles/r02_flops_per_eval_c4.txt). Updated when the kernel changes.
ORD_FP64_FLOPS_PER_EVAL = 1946.9
# the same count in FP64 pipe issue slots (DFMA + DMUL + DADD warp-lane instructions per evaluation): a DMUL or
# DADD takes the slot a DFMA does, so the pipe-slot fraction reads higher than the flop fraction
ORD_FP64_INSTR_PER_EVAL = 1242.8
DIFF_BYTES_PER_NODE_SUBSTEP = 96.0  # 2D stencil: V in + out, 9 coefficients, dt/m


# Problem constants of the reference arm, restated so that arm never imports
# the product package (tests/test_bench_host.py checks them against problems.py).
C1_AMPLITUDE = 592.0   # 2 x the reference's diastolic threshold on the C1 line (296 mV/ms)
C2_AMPLITUDE = 100.0
C2_RADIUS = 0.15
SLAB_AMPLITUDE = 150.0  # C4 endocardial face stimulus, 1 ms
C5_AMPLITUDE, C5_SITE_RADIUS = 450.0, 0.2  # C5 endocardial sites (problems.py C5_*)


def host_cpu():
    """(physical cores available to this process, logical CPUs, CPU model) from /proc/cpuinfo."""
    allowed = os.sched_getaffinity(0)
    cores, model, cpu, phys, core = set(), "unknown", None, None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f.read().splitlines() + [""]:
                if not line.strip():
                    if cpu is not None and cpu in allowed:
                        cores.add((phys, core if core is not None else cpu))
                    cpu, phys, core = None, None, None
                    continue
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "processor":
                    cpu = int(v)
                elif k == "physical id":
                    phys = v
                elif k == "core id":
                    core = v
                elif k == "model name":
                    model = v
    except OSError:
        pass
    return max(1, len(cores) or len(allowed)), len(allowed), model


def pin_openmp(threads):
    """OpenMP placement for the CPU legs; must run before the oracle/reference library is loaded."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    os.environ["OMP_PROC_BIND"] = "close"
    os.environ["OMP_PLACES"] = "cores"


def diffusion_launches(count, fuse):
    """Launches enqueue_diffusion (cwg_host.cu) uses for `count` sub-steps when
    up to `fuse` are fused per launch."""
    return -(-count // fuse)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_problem(config, world, rank, scaling="strong"):
    from paper_2011_04747_b200 import problems
    if config == "c4" and (world == 1 or scaling == "strong"):
        return problems.c4()  # N > 1: every rank gets the full grid and keeps its own y-slab (cwg_slab_plan)
    if config == "c5" and (world == 1 or scaling == "strong"):
        return problems.c5()  # BASELINE configs[4]: the 201M-node slab partitioned across the ranks' y-slabs
    if config == "c2":
        if world == 1:
            return problems.c2()
        # weak scaling: stack world C2-sized blocks in y (one 201-row slab per rank)
        import math as _m
        from paper_2011_04747_b200 import api
        sh = api.Sheet(5.0, 5.0 * world, 0.025, _m.pi / 4, d0_myocyte=0.0012, rho=0.25)
        nodes = sh.select("disc", cx=0.0, cy=0.0, radius=problems.C2_RADIUS)
        cfg = api.SchemeConfig(dt_ms=0.1, t_end_ms=500.0, k0_up=5, k0_down=3)
        return problems.Problem("C2xN", sh, ["ohara2011-epi"], np.zeros(sh.n, np.uint8),
                                [(nodes, 0.0, 1.0, problems.C2_AMPLITUDE, None)], cfg,
                                [sh.nearest(0.0, 0.0), sh.nearest(2.5, 2.5)])
    if config == "c1":
        return problems.c1()
    if config == "c3":
        return problems.c3()
    if config in ("c4", "c5"):
        # weak scaling: the slab grows in y with the number of ranks (same y extent per GPU)
        if config == "c4":
            return problems.slab(5.0, 5.0 * world, 1.0, 0.02, t_end=500.0)
        return problems.slab(10.0, 10.0 * world, 2.0, 0.01, t_end=5.0, stim="sites", n_sites=16 * world,
                             amplitude=problems.C5_AMPLITUDE, site_radius=problems.C5_SITE_RADIUS)
    raise SystemExit(f"unknown config {config}")


def config_block(config, prob, world, l):
    names = {"c2": "BASELINE configs[1]: 2D anisotropic sheet 5x5 cm, 201x201 nodes, fibres 45 deg, "
                   "corner stimulus, ORd-epi, DAETI dt 0.1 ms, 500 ms",
             "c1": "BASELINE configs[0]: 2D isotropic 1x1 cm, 101x101 nodes, ORd-epi, left-edge 2x threshold",
             "c3": "BASELINE configs[2] (extension): 1001x1001 scar/border-zone sheet",
             "c4": "BASELINE configs[3] (extension): 3D slab 5x5x1 cm, 251x251x51 nodes (3,213,051), fibres +60..-60 "
                   "deg, endocardial face stimulus, ORd-epi, DAETI dt 0.1 ms, 500 ms",
             "c5": "BASELINE configs[4] (extension): 3D slab 10x10x2 cm, 1001x1001x201 nodes (201M; y-slabs "
                   "across the ranks), 16 random endocardial sites, ORd-epi"}
    return {"workload": names[config], "nodes": int(prob.n), "nodes_per_gpu": int(prob.n // max(world, 1)),
            "cell_model": prob.models[0], "scheme": "DAETI", "dt_ms": prob.cfg.dt_ms, "k0_up": prob.cfg.k0_up,
            "k0_down": prob.cfg.k0_down, "diffusion_substeps_per_step": 2 * l,
            "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": f"y-slab x{world}" if world > 1 else "single GPU",
            "data": "synthetic tissue (no dataset exists); random-free except the seeded std::mt19937_64 draws of C3/C5"}


def oracle_slab(config):
    """C4 / C5 for the CPU legs on the oracle alone (no product import): the structured slab operator
    (orapy.Slab3DOp, the oracle's own assembly), face / seeded-site endocardial stimulus, ORd-epi."""
    import orapy
    if config == "c4":
        op = orapy.Slab3DOp(250, 250, 50, 0.02)
        iy, ix = np.meshgrid(np.arange(op.ny1), np.arange(op.nx1), indexing="ij")
        nodes = np.sort(op.index(ix, iy, 0).ravel())
        t_end = 500.0
    else:
        # c5: a y-sub-slab of the 1001 x 1001 x 201 grid (y <= 0.2 cm, 1001 x 21 x 201 = 4.2M nodes: the
        # full slab's state alone is ~70 GB of host memory) with the full slab's 16 seeded sites
        # (problems.site_centers: std::mt19937_64(2011)); node-updates/s is a per-node rate
        op = orapy.Slab3DOp(1000, 20, 200, 0.01)
        u = orapy.uniform_mt64(2011, 32, 0.0, 1.0)
        iy, ix = np.meshgrid(np.arange(op.ny1), np.arange(op.nx1), indexing="ij")
        x, y = ix * op.h, iy * op.h
        sel = np.zeros(ix.shape, bool)
        for k in range(16):
            sel |= np.sqrt((x - 10.0 * u[2 * k]) ** 2 + (y - 10.0 * u[2 * k + 1]) ** 2) <= C5_SITE_RADIUS + 1e-9
        nodes = np.sort(op.index(ix[sel], iy[sel], 0))
        t_end = 5.0
    return op, nodes, t_end


def slab_amplitude(config):
    return SLAB_AMPLITUDE if config == "c4" else C5_AMPLITUDE


def cpu_reference_steps(config, steps, warmup, budget_s, threads):
    """Time the reference's own StrangIntegrator::advance (oracle/_ref/libcwref.so) on host cores -- or,
    for the configurations the reference cannot express (C4, C5), the oracle's restatement of it."""
    pin_openmp(threads)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    if config in ("c4", "c5"):
        import orapy
        op, nodes, t_end = oracle_slab(config)
        it = orapy.Integrator(op, op.dt_s, ["ohara2011-epi"], np.zeros(op.n, np.uint8),
                              [(nodes, 0.0, 1.0, slab_amplitude(config), None)], scheme="DAETI", dt=0.1, k0_up=5,
                              k0_down=3)
        n_total = int(round(t_end / 0.1))
        for st in range(warmup):
            it.advance(st * 0.1, st, n_total)
        kh0 = it.khist.copy()
        t0 = time.perf_counter()
        done = 0
        for st in range(warmup, min(warmup + steps, n_total)):
            it.advance(st * 0.1, st, n_total)
            done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        wall = time.perf_counter() - t0
        evals = int(np.sum((it.khist - kh0) * np.arange(len(it.khist))))
        diff = done * it.n * 2 * it.l
        return {"steps": done, "wall_s": wall, "evals": evals, "diff": diff, "n": it.n, "l": it.l,
                "value": (evals + diff) / wall, "sim_ms_per_s": done * 0.1 / wall, "kind": "port",
                "what": "oracle restatement of StrangIntegrator::advance (oracle/cw_oracle.c, OpenMP)"}
    import refpy
    if config == "c2":
        p = refpy.Sheet(5.0, 5.0, 0.025, math.pi / 4, d0=0.0012, rho=0.25)
        nodes = p.select("disc", cx=0.0, cy=0.0, radius=C2_RADIUS)
        amp, t_end = C2_AMPLITUDE, 500.0
    elif config == "c1":  # BASELINE configs[0]: 1 x 1 cm isotropic, left-edge line at 2x threshold, 400 ms
        p = refpy.Sheet(1.0, 1.0, 0.01, 0.0, d0=0.001, rho=1.0)
        nodes = p.select("x_le", value=0.0)
        amp, t_end = C1_AMPLITUDE, 400.0
    else:
        raise SystemExit("reference arm implemented for c1, c2, c4 and c5")
    p.set_models(["ohara2011-epi"])
    p.add_stimulus(nodes, 0.0, 1.0, amp)
    p.init_state()
    n_total = int(round(t_end / 0.1))
    p.integrator(scheme="DAETI", dt=0.1, t_end=t_end, k0_up=5, k0_down=3, workers=threads)
    for s in range(warmup):
        p.advance(s * 0.1, s, n_total)
    kh0 = p.integrator_khist().copy()
    t0 = time.perf_counter()
    done = 0
    for s in range(warmup, min(warmup + steps, n_total)):  # a fast host may finish the run within the budget
        p.advance(s * 0.1, s, n_total)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    wall = time.perf_counter() - t0
    kh1 = p.integrator_khist()
    evals = int(np.sum((kh1 - kh0) * np.arange(len(kh1))))
    diff = done * p.n * 2 * p.l
    return {"steps": done, "wall_s": wall, "evals": evals, "diff": diff, "n": p.n, "l": p.l,
            "value": (evals + diff) / wall, "sim_ms_per_s": done * 0.1 / wall, "kind": "reference",
            "what": "cardwave::StrangIntegrator::advance (oracle/_ref/libcwref.so, unmodified reference)"}


WORKLOAD = {"c1": "C1 (BASELINE configs[0])", "c2": "C2 (BASELINE configs[1])",
            "c4": "C4 (BASELINE configs[3], 251x251x51 slab)", "c5": "C5 (BASELINE configs[4], 1001x1001x201 slab)"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads, logical, model = host_cpu()
    r = cpu_reference_steps(args.config, args.steps, args.warmup, args.ref_budget, threads)
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["wall_s"] * 1e3 / max(r["steps"], 1),
            "higher_is_better": True, "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config] + " through " + r["what"],
                       "nodes": r["n"], "threads": threads, "cpu_model": model, "logical_cpus": logical,
                       "omp": "OMP_PROC_BIND=close OMP_PLACES=cores"},
            "sim_ms_per_s": r["sim_ms_per_s"],
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": r["kind"],
                             "cpu_model": model,
                             "sample": f"{args.config.upper()} outer steps {args.warmup}..{args.warmup + r['steps']} "
                                       f"({r['steps']} x 0.1 ms) after {args.warmup} warm-up steps, "
                                       f"OpenMP {threads} threads on physical cores ({logical} logical CPUs), "
                                       f"{r['what']}"},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c4", "c1", "c2", "c3", "c5"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1 with --config c4: split one C4 grid (strong) or one C4 per rank (weak)")
    ap.add_argument("--ref-budget", type=float, default=20.0, help="seconds of reference CPU work per arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        if args.steps is None:
            args.steps = 200
        return run_reference_arm(args)

    import torch
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None

    def new_nccl_id():
        """A fresh ncclUniqueId from rank 0 for every communicator (an id
        bootstraps exactly one communicator); gloo carries the 128 bytes."""
        obj = [b""]
        if rank == 0:
            import ctypes
            nc = ctypes.CDLL("libnccl.so.2")  # the torch-bundled NCCL (plumbing only)
            buf = (ctypes.c_ubyte * 128)()
            assert nc.ncclGetUniqueId(buf) == 0
            obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        nccl_id = new_nccl_id()

    prob = build_problem(args.config, world, rank, args.scaling)
    setup = prob.setup()
    n_total = int(math.ceil(prob.cfg.t_end_ms / prob.cfg.dt_ms - 1e-9))
    if args.steps is None:
        args.steps = n_total - args.warmup
    if args.warmup + args.steps > n_total:  # extend the simulated window to fit
        prob.cfg.t_end_ms = (args.warmup + args.steps) * prob.cfg.dt_ms
    integ = cw.StrangIntegrator(setup, prob.cfg, model_of_node=prob.model_of_node, device=local, rank=rank,
                                world=world, nccl_id=nccl_id)
    info = integ.info
    big = prob.n > 20_000_000
    if big:  # 10^8 nodes: make_initial_state on the device (the AoS host copy would be ~64 GB)
        integ.init_rest()
    else:
        integ.upload(prob.initial_state())
    integ.run_begin()
    integ.run_steps(0, args.warmup)
    integ.run_sync()
    torch.cuda.synchronize()

    K = args.steps
    step_ms, react_ms, diff_ms = np.zeros(K), np.zeros(K), np.zeros(K)
    lib = L.lib()
    ev0 = lib.cwg_reaction_evals(integ._h)
    launches0 = integ.launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    with ClockSampler(local) as clocks:
        rc = lib.cwg_bench_steps(integ._h, args.warmup, K, FLUSH_BYTES, 0, L.dp(step_ms), L.dp(react_ms),
                                 L.dp(diff_ms))
        torch.cuda.synchronize()
    if rc != 0:
        raise SystemExit(f"cwg_bench_steps failed ({rc}): {lib.cwg_last_error().decode()}")
    if dist:
        dist.barrier()
    wall = time.perf_counter() - t_wall0
    integ.run_sync()  # surfaces an InstabilityError from the timed window
    ev1 = lib.cwg_reaction_evals(integ._h)
    launches = integ.launch_count() - launches0
    t_dev_ms = float(step_ms.sum())
    if dist:
        tt = torch.tensor([t_dev_ms], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev_ms = float(tt.item())
    reaction_evals = ev1 - ev0  # global (khist all-reduced)
    diff_updates = prob.n * 2 * info.l * K
    value = (reaction_evals + diff_updates) / (t_dev_ms / 1e3)

    # --- roofline of the dominant kernel (ORd reaction): FP64 pipe
    peaks, peak_src = load_peaks()
    fp64_peak = lib.cwg_fp64_peak_tflops(local, 0.5)
    local_evals = reaction_evals / world
    react_tot_ms = float(react_ms.sum())
    achieved = ORD_FP64_FLOPS_PER_EVAL * local_evals / (react_tot_ms / 1e3) / 1e12
    traffic, pipe_ncu = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            summ = json.load(f)
        # DRAM bytes per reaction launch from the ncu capture of the same configuration (C4; other configs: none)
        traffic = summ.get("react_c4", {}).get("dram_bytes_per_launch") if args.config == "c4" else None
        pipe = summ.get("fp64_pipe_active_pct_of_active", {})
        pipe_ncu = pipe.get("c2_latency_shape" if args.config in ("c1", "c2") else "c4_throughput_shape")
    except (OSError, ValueError):
        pass
    diff_tot_ms = float(diff_ms.sum())
    is3d = args.config in ("c4", "c5")
    # Algorithmic diffusion bytes per step: every launch reads V and writes V
    # once per node (16 B) plus the node's coefficients -- 80 B of per-node
    # arrays in 2D, 0 for the cached 3D structured tables; a launch fusing T
    # sub-steps counts once (fused-traffic bound).
    # large one-GPU 2D sheets run the TMA-fed persistent kernel (cwg_host.cu enqueue_diffusion), which
    # fuses up to 6 sub-steps per launch; the register-loading kernel up to 4
    sheet = getattr(prob, "sheet", None)
    tma_path = (not is3d and world == 1 and sheet is not None and os.environ.get("CWG_TB_TMA", "1") != "0"
                and -(-sheet.nx1 // 64) * -(-sheet.ny1 // 16) >= 2 * 148)
    cap = 6 if tma_path else 4
    fuse = 1 if is3d else int(os.environ.get("CWG_DIFF_TB", str(cap)))
    fuse = max(1, min(cap, fuse))  # (multi-rank 2D: halo depth min(4, rows per rank) >= 4 in every bench config)
    launches_per_step = diffusion_launches(2 * info.l, fuse)
    coef_b = 0.0 if is3d else 80.0
    diff_bytes_step = info.n_local * launches_per_step * (16.0 + coef_b)
    diff_bytes = diff_bytes_step / (info.n_local * 2 * info.l)
    diff_gbs = diff_bytes_step * K / (diff_tot_ms / 1e3) / 1e9

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": t_dev_ms / K, "higher_is_better": True,
            "scaling": "strong" if (args.config in ("c4", "c5") and args.scaling == "strong") else "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_block(args.config, prob, world, info.l),
            "sim_ms_per_s": K * prob.cfg.dt_ms / (t_dev_ms / 1e3),
            "reaction_node_updates_per_s": reaction_evals / (t_dev_ms / 1e3),
            "diffusion_node_updates_per_s": diff_updates / (t_dev_ms / 1e3),
            "mean_k": reaction_evals / (prob.n * K),
            "phase_ms": {"reaction": react_tot_ms / K, "diffusion_and_record": diff_tot_ms / K},
            "wall_s_timed_region": wall,
            "roofline": {"bound": "fp64", "kernel": "react_kernel<ModelOrd<epi>>", "achieved": achieved,
                         "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak if fp64_peak > 0 else None,
                         "traffic": traffic, "peak_source": "in-run DFMA microbenchmark (MEASURED_PEAKS.json has no "
                                                             "FP64 entry)",
                         "flops_per_eval": ORD_FP64_FLOPS_PER_EVAL,
                         "fp64_instr_per_eval": ORD_FP64_INSTR_PER_EVAL,
                         "fp64_pipe_slot_frac": (ORD_FP64_INSTR_PER_EVAL * local_evals / (react_tot_ms / 1e3) / 1e12)
                                                / (fp64_peak / 2.0) if fp64_peak > 0 else None,
                         "fp64_pipe_active_ncu": pipe_ncu / 100.0 if pipe_ncu is not None else None,
                         "note": ("latency regime: ~1 node per lane (8 warps/SM at >168 registers), each node's k "
                                  "sub-steps sequential, so the step's largest k sets the critical path; the "
                                  "event-timed phase includes ~10 us of launch/completion latency around a ~42 us "
                                  "kernel span (tools/react_trace.py, DESIGN.md 3.5)" if args.config in ("c1", "c2") else
                                  "throughput regime: one 384-thread lockstep block per SM; FP64 pipe 52% of "
                                  "active cycles on C4, 8-cycle FP64 latency with 3 warps per sub-partition "
                                  "(profiles/r02g_react_c4_digest.txt, r02_fp64_latency.txt); traffic = ncu DRAM "
                                  "read+write per launch (algorithmic 677 B x 3.2M nodes = 2.18 GB)")},
            "roofline_diffusion": {"bound": "hbm",
                                   "kernel": "diffuse_struct3d" if is3d else (
                                       ("diffuse_stencil2d_tbm (TMA)" if tma_path else "diffuse_stencil2d_tb")
                                       if fuse > 1 and launches_per_step < 2 * info.l else "diffuse_stencil2d"),
                                   "achieved": diff_gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                   "frac": diff_gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                                   "peak_source": peak_src, "bytes_per_node_substep": diff_bytes,
                                   "launches_per_step": launches_per_step,
                                   # the bit-exact row sum is 28 DMUL + 28 DADD per node-substep (27-point 3D /
                                   # 10 + 10 in 2D): against 16 B of V the 3D kernel is FP64-bound, so its FP64
                                   # fraction is reported beside the HBM one
                                   "fp64_ops_per_node_substep": 56 if is3d else 20,
                                   "fp64_tflops": (56 if is3d else 20) * info.n_local * 2 * info.l * K
                                                  / (diff_tot_ms / 1e3) / 1e12,
                                   "fp64_frac": ((56 if is3d else 20) * info.n_local * 2 * info.l * K
                                                 / (diff_tot_ms / 1e3) / 1e12 / fp64_peak) if fp64_peak > 0 else None,
                                   "note": "phase time includes probe/detector recording and the ~6 us that any "
                                           "kernel between two CUDA events costs here (DESIGN.md 3.5)"},
            "clocks": clocks.summary(), "gpu_launches": int(launches),
            "launch_mode": "one CUDA graph per step (event-record nodes at step start / after reaction / end)",
            "ord_launch_shape": ("2 x 128-thread free-running blocks per SM, 254 registers (latency regime)"
                                 if args.config in ("c1", "c2") else
                                 "one 384-thread lockstep block per SM, 168 registers (throughput regime)")}

    # --- end to end through the public API (run_simulation) with pinned host state
    if big:
        line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                       "note": "skipped: host AoS state of a 10^8-node slab is ~64 GB"}
    if not args.no_e2e and not big:
        pin = lambda a: (lambda t: (t.copy_(torch.from_numpy(a)), t.numpy())[1])(
            torch.empty(a.shape, dtype=torch.float64, pin_memory=True))
        st0 = prob.initial_state()
        st0.v, st0.s, st0.last_dvdt = pin(st0.v), pin(st0.s), pin(st0.last_dvdt)
        # the result lands in pinned host buffers too (allocated once, outside the timed region)
        fin = st0.copy()
        fin.v, fin.s, fin.last_dvdt = pin(fin.v), pin(fin.s), pin(fin.last_dvdt)
        pinned = lambda dt: torch.empty(prob.n, dtype=dt, pin_memory=True).numpy()
        maps_out = tuple(cw.ScalarMap(pinned(torch.float64), pinned(torch.bool)) for _ in range(2))
        e2e_cfg = cw.SchemeConfig(scheme=prob.cfg.scheme, dt_ms=prob.cfg.dt_ms,
                                  t_end_ms=(args.warmup + K) * prob.cfg.dt_ms, k0_up=prob.cfg.k0_up,
                                  k0_down=prob.cfg.k0_down)
        # three back-to-back calls, median reported (host-side setup jitter); each call
        # builds its own integrator, as the reference's run_simulation does
        walls, creates = [], []
        for _rep in range(3):
            e_id = new_nccl_id() if dist else None
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e_integ = cw.StrangIntegrator(setup, e2e_cfg, model_of_node=prob.model_of_node, device=local, rank=rank,
                                          world=world, nccl_id=e_id)
            creates.append(time.perf_counter() - t0)
            res = cw.run_simulation(st0, setup, e2e_cfg, device=local, integrator=e_integ, final_state_out=fin,
                                  maps_out=maps_out)
            torch.cuda.synchronize()
            w_s = time.perf_counter() - t0
            if dist:
                tt = torch.tensor([w_s], dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                w_s = float(tt.item())
            walls.append(w_s)
            e_integ.close()  # run_simulation leaves st0 untouched: the next call starts from the same state
        e2e_s = float(np.median(walls))
        n_steps_e = args.warmup + K
        e_evals = int(np.sum(res.k_histogram * np.arange(len(res.k_histogram))))
        e_val = (e_evals + prob.n * 2 * info.l * n_steps_e) / e2e_s
        stride = st0.stride
        h2d = prob.n * (2 + stride) * 8
        d2h = prob.n * (2 + stride) * 8 + prob.n * (2 * 8 + 2) + len(prob.probes) * info.n_samples * 8
        line["e2e"] = {"value": e_val, "unit": UNIT, "h2d_bytes_per_step": h2d / n_steps_e,
                       "d2h_bytes_per_step": d2h / n_steps_e,
                       "call": "paper_2011_04747_b200.run_simulation (cwg_create + state upload from pinned host "
                               "memory + all steps + traces/LAT/APD maps/final-state download into pinned host memory)",
                       "steps": n_steps_e, "wall_s": e2e_s, "wall_s_all": walls,
                       "create_s_all": creates}

    # --- CPU baseline: the reference itself on this host (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in ("c1", "c2", "c4", "c5"):
        threads, logical, model = host_cpu()
        try:
            r = cpu_reference_steps(args.config, 100000, args.warmup, 15.0, threads)
            line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": r["kind"],
                                    "cpu_model": model,
                                    "sample": f"{args.config.upper()} outer steps {args.warmup}.."
                                              f"{args.warmup + r['steps']} ({r['n']} nodes) through {r['what']}, "
                                              f"~15 s budget, OpenMP {threads} threads on physical cores "
                                              f"({logical} logical CPUs, OMP_PROC_BIND=close)",
                                    "sim_ms_per_s": r["sim_ms_per_s"]}
        except Exception as e:  # the checker library is a build artefact; report its absence
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    integ.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
