#!/bin/bash
# Round-2 (second session) profiling on one B200: full bench lines, the ncu launch list of the default (C4)
# bench, one full ncu capture of the reaction kernel (C4) and of the 2D register-quad diffusion kernel (C3),
# and the host-vs-device assembly timing. Outputs -> gpurun_out/r02b/.
set -u
O=gpurun_out/r02b
mkdir -p $O
for c in ${CONFIGS:-c4 c3}; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python tools/assembly_timing.py > $O/assembly_c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:react_kernel -s 3 -c 1 -o $O/react_c4 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_react.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diffuse_stencil2d_tbq -s 8 -c 1 -o $O/tbq_c3 \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_tbq.log 2>&1
echo done
