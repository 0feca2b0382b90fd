#!/bin/bash
# Round profiling on one B200 (run through gpurun): bench lines for every BASELINE config, the ncu launch
# list of the default (C4) bench, and one full ncu capture of the two dominant kernels. Outputs -> gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
for c in c4 c3 c2 c1 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:react_kernel -s 3 -c 1 -o $O/react_c4 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_react.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diffuse_struct3d -s 4 -c 1 -o $O/s3_c4 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_s3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diffuse_stencil2d_tbm -s 8 -c 1 -o $O/tbm_c3 \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_tbm.log 2>&1
echo done
