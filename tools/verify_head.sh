#!/bin/bash
# Quick validation of the current build on one B200: GPU suite, smoke, default C4 bench and the driver's short run.
set -u
O=gpurun_out/${1:-head}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_c4_short.json 2> $O/bench_c4_short.err
echo done
