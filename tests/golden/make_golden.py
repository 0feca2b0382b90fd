"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libcwref.so).

Run in the build container (needs /root/reference compiled by `make -C oracle ref`):
    python tests/golden/make_golden.py
The fixtures pin the C restatement oracle (tests/test_golden.py) on machines
where the reference cannot be built. Reference sources are not copied; only
numeric outputs of the reference library are stored.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import refpy  # noqa: E402

MODELS = ["aliev-panfilov", "ohara2011-endo", "ohara2011-epi", "ohara2011-mid", "maccannell2007"]


def rates_fixture():
    rng = np.random.default_rng(20110474)
    out = {}
    for m in MODELS:
        ns, ss, rest = refpy.model_info(m)
        n = 64
        if m == "aliev-panfilov":
            v = rng.uniform(-85, 25, n)
            s = rng.uniform(0, 2, (n, ns))
        else:
            v = rng.uniform(-95, 45, n)
            s = np.tile(rest[1:], (n, 1)) * rng.uniform(0.7, 1.3, (n, ns))
        v[0] = rest[0]
        s[0] = rest[1:]
        ist = rng.choice([0.0, 80.0], n)
        dv, ds = refpy.rates(m, v, s, ist)
        key = m.replace("-", "_")
        out.update({f"{key}_v": v, f"{key}_s": s, f"{key}_ist": ist, f"{key}_dv": dv, f"{key}_ds": ds,
                    f"{key}_rest": rest, f"{key}_stable_step": np.array([ss])})
    np.savez_compressed(os.path.join(HERE, "rates.npz"), **out)


def rules_fixture():
    rng = np.random.default_rng(7)
    rows = []
    for _ in range(500):
        d = float(rng.choice([-1, 1]) * 10 ** rng.uniform(-3, 2.5))
        sch = int(rng.integers(3))
        k0d = int(rng.integers(1, 4))
        k0u = k0d + int(rng.integers(0, 5))
        km = int(rng.integers(1, 20))
        k = refpy.reaction_substeps(d, ["OST", "OSTAR", "DAETI"][sch], k0u, k0d, km)
        dt, dts = float(rng.uniform(0.005, 0.5)), float(rng.uniform(0.001, 0.3))
        strict = int(rng.integers(2))
        l, dt_ad = refpy.diffusion_substeps(dt, dts, strict, ["OST", "OSTAR", "DAETI"][sch])
        rows.append((d, sch, k0u, k0d, km, k, dt, dts, strict, l, dt_ad))
    np.savez_compressed(os.path.join(HERE, "rules.npz"), rows=np.array(rows, dtype=np.float64))


def runs_fixture():
    out = {}
    # C1 sheet, Aliev-Panfilov, x <= 0.05 strip at 100 mV/ms, DAETI dt 0.1, 40 ms (bit-exact everywhere)
    s = refpy.Sheet(1, 1, 0.01, 0.0, d0=0.001, rho=1.0)
    nodes = s.select("x_le", value=0.05)
    s.set_models(["aliev-panfilov"])
    s.add_stimulus(nodes, 0.0, 1.0, 100.0)
    s.init_state()
    r = s.run(scheme="DAETI", dt=0.1, t_end=40.0, k0_down=1, probes=[0, 5050, 10200])
    out.update(ap_v=r["state"][0], ap_s=r["state"][1], ap_khist=r["k_histogram"], ap_lat=r["lat"],
               ap_lat_valid=r["lat_valid"], ap_traces=np.array([tv[1] for tv in r["traces"]]))
    # C1 sheet, ORd-epi, left edge 592 mV/ms, k0_down 3, 5 ms
    s = refpy.Sheet(1, 1, 0.01, 0.0, d0=0.001, rho=1.0)
    nodes = s.select("x_le", value=0.0)
    s.set_models(["ohara2011-epi"])
    s.add_stimulus(nodes, 0.0, 1.0, 592.0)
    s.init_state()
    r = s.run(scheme="DAETI", dt=0.1, t_end=5.0, k0_down=3, probes=[0, 5050, 10200])
    out.update(ord_v=r["state"][0], ord_khist=r["k_histogram"], ord_traces=np.array([tv[1] for tv in r["traces"]]))
    # the abort fixture: paper k0 (k0_down = 1)
    s = refpy.Sheet(1, 1, 0.01, 0.0, d0=0.001, rho=1.0)
    s.set_models(["ohara2011-epi"])
    s.add_stimulus(nodes, 0.0, 1.0, 592.0)
    s.init_state()
    try:
        s.run(scheme="DAETI", dt=0.1, t_end=5.0, k0_down=1)
        raise SystemExit("expected the reference to abort")
    except refpy.RefError as e:
        out.update(abort_node=np.array([e.node]), abort_t=np.array([e.t]))
    # dt_s of the survey's geometries
    out["dt_s"] = np.array([refpy.Sheet(1, 1, 0.01, 0.0, d0=0.001, rho=1.0).dt_s,
                            refpy.Sheet(5, 5, 0.025, np.pi / 4, d0=0.0012, rho=0.25).dt_s,
                            refpy.Sheet(1, 1, 0.01, 0.0, d0=0.0017, rho=0.25).dt_s])
    # diastolic_threshold on two small sheets
    thr = []
    for (lx, ly, h, model, strip, window) in [(1.5, 0.3, 0.05, "aliev-panfilov", 0.1, 200.0),
                                              (1.2, 0.2, 0.04, "ohara2011-epi", 0.08, 40.0)]:
        p = refpy.Sheet(lx, ly, h, 0.0, d0=0.0017, rho=1.0)
        thr.append(p.threshold(model, p.select("x_le", value=strip), window_ms=window))
    out["thresholds"] = np.array(thr)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)


PACE_CASES = [("aliev-panfilov", 500.0, 3, 0.5, 1.0), ("maccannell2007", 400.0, 2, 10.0, 1.0),
              ("ohara2011-endo", 300.0, 2, 80.0, 1.0), ("ohara2011-epi", 400.0, 3, 60.0, 0.5),
              ("ohara2011-mid", 250.0, 2, 80.0, 1.0)]


def pace_fixture():
    """cardwave::pace_to_steady_state (ionic.cpp:122-165) outputs + one |V| > 1000 abort."""
    out = {}
    for i, (m, cl, nb, amp, dur) in enumerate(PACE_CASES):
        st, mr, apd = refpy.pace(m, cl, nb, amp, dur)
        out.update({f"c{i}_state": st, f"c{i}_max_rel": np.array([mr]), f"c{i}_apd": apd})
    try:
        refpy.pace("ohara2011-epi", 300.0, 2, 3000.0, 2.0)
        out["abort_t"] = np.array([np.nan])
    except refpy.RefError as e:
        out["abort_t"] = np.array([e.t])
    np.savez_compressed(os.path.join(HERE, "pace.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rates", "rules", "runs", "pace"]
    for name in which:
        globals()[name + "_fixture"]()
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))
