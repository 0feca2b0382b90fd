"""Executed FP64 flops per ORd rates evaluation, for bench.py's roofline.

Run under ncu so that every reaction launch is counted:
  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
      -k regex:react_kernel --csv --log-file gpurun_out/flops.csv python tools/flops_per_eval.py [c2|c4] [steps]
then: python tools/flops_per_eval.py --parse gpurun_out/flops.csv gpurun_out/evals.txt
"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out="gpurun_out/evals.txt", steps=60, config="c2"):
    import paper_2011_04747_b200 as cw
    from paper_2011_04747_b200 import problems, _lib as L
    p = {"c2": problems.c2, "c4": problems.c4}[config](t_end=steps * 0.1)
    integ = cw.StrangIntegrator(p.setup(), p.cfg, model_of_node=p.model_of_node)
    integ.upload(p.initial_state())
    integ.run_begin()
    integ.run_steps(0, integ.info.n_steps)
    integ.run_sync()
    evals = int(L.lib().cwg_reaction_evals(integ._h))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    open(out, "w").write(f"{evals}\n")
    print("evals", evals)


def parse(csv_path, evals_path):
    tot = {"dfma": 0.0, "dmul": 0.0, "dadd": 0.0}
    lines = [l for l in open(csv_path) if l.startswith('"')]
    for row in csv.DictReader(lines):
        for k in tot:
            if row.get("Metric Name", "").endswith(f"op_{k}_pred_on.sum"):
                tot[k] += float(row["Metric Value"].replace(",", ""))
    evals = int(open(evals_path).read().split()[0])
    flops = 2 * tot["dfma"] + tot["dmul"] + tot["dadd"]
    print({k: v / evals for k, v in tot.items()}, "flops/eval", flops / evals)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--parse":
        parse(sys.argv[2], sys.argv[3])
    else:  # [config (c2 | c4)] [steps]
        run(config=sys.argv[1] if len(sys.argv) > 1 else "c2", steps=int(sys.argv[2]) if len(sys.argv) > 2 else 60)
