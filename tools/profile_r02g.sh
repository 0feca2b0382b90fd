#!/bin/bash
# Round-2 final-build evidence (the r02e / r02f / r02g passes of the last session ran this script) on one B200: GPU test suite, bench lines for every BASELINE config, the C4
# reference arm, executed FP64 flops per evaluation (C4, C2), the ncu launch list of the default bench and one
# full ncu capture of the reaction kernel. Outputs -> gpurun_out/r02g/.
set -u
O=gpurun_out/r02g
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c4 c3 c2 c1 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_c4_short.json 2> $O/bench_c4_short.err
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for c in c4 c2; do
  timeout 900 ncu --metrics $M -k regex:react_kernel --csv --log-file $O/flops_$c.csv \
    python tools/flops_per_eval.py $c 40 > $O/flops_$c.log 2>&1
  cp gpurun_out/evals.txt $O/evals_$c.txt
  python tools/flops_per_eval.py --parse $O/flops_$c.csv $O/evals_$c.txt > $O/flops_$c.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:react_kernel -s 3 -c 1 -o $O/react_c4 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_react.log 2>&1
timeout 300 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diffuse_struct3d -s 4 -c 1 -o $O/struct3d_c4 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_struct3d.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 300 python tools/refill_cost_probe.py 12 > $O/refill_cost_probe.txt 2>&1
echo done
