"""Shared helpers: run a Problem on the GPU (product) and on the oracle (checker)."""
import numpy as np


def csr_of(problem):
    op = problem.sheet.op
    return (op.row_ptr, op.col, op.val, op.lumped_mass)


def gpu_run(problem, device=0):
    import paper_2011_04747_b200 as cw
    st = problem.initial_state()
    return cw.run_simulation(st, problem.setup(), problem.cfg, device=device)


def oracle_run(problem, **over):
    import orapy
    cfg = problem.cfg
    kw = dict(scheme=cfg.scheme.name, dt=cfg.dt_ms, t_end=cfg.t_end_ms, k0_up=cfg.k0_up, k0_down=cfg.k0_down,
              strict=cfg.strict_substeps, record_interval=cfg.record_interval_ms, probes=problem.probes,
              gkr_scale=problem.gkr_scale)
    kw.update(over)
    return orapy.run_simulation(csr_of(problem), problem.sheet.op.dt_s, problem.models, problem.model_of_node,
                                problem.stimuli, **kw)


def lat_order_equal(lat_a, valid_a, lat_b, valid_b, nx1):
    """LAT rank order on the sampled node set (every 10th node per axis), ties by node index."""
    n = len(lat_a)
    ny1 = n // nx1
    ys, xs = np.meshgrid(np.arange(0, ny1, 10), np.arange(0, nx1, 10), indexing="ij")
    idx = (ys * nx1 + xs).ravel()
    if not np.array_equal(valid_a[idx], valid_b[idx]):
        return False
    sel = idx[valid_a[idx]]
    oa = sel[np.lexsort((sel, lat_a[sel]))]
    ob = sel[np.lexsort((sel, lat_b[sel]))]
    return np.array_equal(oa, ob)
