#!/bin/bash
# Bench lines of every BASELINE config + the C4 reference arm + the driver's short run -> gpurun_out/$1/
set -u
O=gpurun_out/${1:-lines}
mkdir -p $O
for c in c4 c3 c2 c1 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_c4_short.json 2> $O/bench_c4_short.err
echo done
