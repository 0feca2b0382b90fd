#!/bin/bash
# A/B of ORd launch shapes (CWG_ORD_VARIANT) on the headline config: parity subset under the first
# non-default variant, then reaction ms per step of each variant, alternated twice.
# usage: tools/ab_variants.sh "1 9" [steps]
VS=$1; STEPS=${2:-300}
mkdir -p gpurun_out
for v in $VS; do
  [ "$v" = 1 ] && continue
  CWG_ORD_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_scale_parity.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
done
for rep in 1 2; do for v in $VS; do
CWG_ORD_VARIANT=$v timeout 600 python bench.py --config c4 --steps $STEPS --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${v}_$rep.log 2>&1
python - gpurun_out/var_${v}_$rep.log $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('variant',sys.argv[2],'react %.4f'%d['phase_ms']['reaction'],'ms/step %.4f'%d['ms_per_step'])
PY
done; done
