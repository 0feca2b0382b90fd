#!/bin/bash
# Re-measure after a reaction-kernel change: executed FP64 flops per evaluation (ncu, C4 and C2), the full C4
# and C3 bench lines, and the ORd-touching GPU tests. Outputs -> gpurun_out/rm/.
set -u
O=gpurun_out/rm
mkdir -p $O
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for c in c4 c2; do
  timeout 900 ncu --metrics $M -k regex:react_kernel --csv --log-file $O/flops_$c.csv \
    python tools/flops_per_eval.py $c 40 > $O/flops_$c.log 2>&1
  cp gpurun_out/evals.txt $O/evals_$c.txt
  python tools/flops_per_eval.py --parse $O/flops_$c.csv $O/evals_$c.txt > $O/flops_$c.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c3 > $O/bench_c3.json 2> $O/bench_c3.err
echo done
