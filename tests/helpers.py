"""Shared helpers: run a Problem on the GPU (product) and on the oracle (checker)."""
import numpy as np


def csr_of(problem):
    op = problem.sheet.op
    if hasattr(op, "s3d"):  # 3D slab: the oracle's own CSR assembly of the same operator
        import orapy
        csr, _ = orapy.assemble_slab3d(op.nx, op.ny, op.nz, op.h, op.d_long, op.rho, op.angles)
        return csr
    return (op.row_ptr, op.col, op.val, op.lumped_mass)


def paced_state(problem):
    """A problem with `pacing` starts its paced model from pace_to_steady_state: both the GPU run and the
    oracle run start from the ORACLE's paced state (ionic.cpp:122-167 restated), so they see the same input."""
    if problem.pacing is None:
        return None
    import orapy
    mid, cl, beats, amp, dur = problem.pacing
    return orapy.pace(problem.models[mid], cl, beats, amp, dur)[0]


def gpu_run(problem, device=0):
    import paper_2011_04747_b200 as cw
    st = problem.initial_state(paced_state=paced_state(problem))
    return cw.run_simulation(st, problem.setup(), problem.cfg, device=device)


def oracle_run(problem, **over):
    import orapy
    cfg = problem.cfg
    kw = dict(scheme=cfg.scheme.name, dt=cfg.dt_ms, t_end=cfg.t_end_ms, k0_up=cfg.k0_up, k0_down=cfg.k0_down,
              strict=cfg.strict_substeps, record_interval=cfg.record_interval_ms, probes=problem.probes,
              gkr_scale=problem.gkr_scale)
    if problem.pacing is not None and "init" not in over:
        st = problem.initial_state(paced_state=paced_state(problem))
        kw["init"] = (st.v, st.s.reshape(problem.n, -1), st.last_dvdt)
    kw.update(over)
    return orapy.run_simulation(csr_of(problem), problem.sheet.op.dt_s, problem.models, problem.model_of_node,
                                problem.stimuli, **kw)


def sampled_nodes(n, nx1, probes=()):
    """every 10th node along each axis plus the probes."""
    ny1 = n // nx1
    ys, xs = np.meshgrid(np.arange(0, ny1, 10), np.arange(0, nx1, 10), indexing="ij")
    return np.union1d((ys * nx1 + xs).ravel(), np.asarray(list(probes), np.int64))


def lat_order_equal(lat_a, valid_a, lat_b, valid_b, nx1, probes=(), tie_ms=1e-9):
    """LAT rank order on the sampled node set, ties (|dLAT| <= tie_ms) broken by node index.

    A planar wave activates whole columns at the same time in exact
    arithmetic; their computed LATs differ by rounding only, so values closer
    than tie_ms are ties. The orders agree iff, walking the nodes in the
    order of lat_a, lat_b never decreases by more than tie_ms (and vice versa).
    """
    idx = sampled_nodes(len(lat_a), nx1, probes)
    if not np.array_equal(valid_a[idx], valid_b[idx]):
        return False
    sel = idx[valid_a[idx]]
    for x, y in ((lat_a, lat_b), (lat_b, lat_a)):
        order = sel[np.lexsort((sel, x[sel]))]
        yy = y[order]
        if np.any(np.maximum.accumulate(yy) - yy > tie_ms):
            return False
    return True


def run_both(problem, **over):
    """(gpu_result | InstabilityError, oracle_result | OracleInstability)."""
    import orapy
    import paper_2011_04747_b200 as cw
    try:
        g = gpu_run(problem)
    except cw.InstabilityError as e:
        g = e
    try:
        o = oracle_run(problem, **over)
    except orapy.OracleInstability as e:
        o = e
    return g, o
