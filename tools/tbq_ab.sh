#!/bin/bash
# A/B of the 2D fused diffusion kernels: register quads (default) vs the slot kernel (CWG_TBQ=0).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_diffusion_tb.py tests/test_gpu_edges.py tests/test_gpu_scale_parity.py -m gpu -q -x > gpurun_out/tbq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tbq_tests.log
for tag in tbm tbq; do
  if [ $tag = tbm ]; then export CWG_TBQ=0; else unset CWG_TBQ; fi
  for c in c2 c3; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$tag.log 2>&1; echo "$c $tag rc=$?"
  done
done
python - <<'PY'
import json
for c in ("c2", "c3"):
    for tag in ("tbm", "tbq"):
        f = f"gpurun_out/ab_{c}_{tag}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(c, tag, "%.4e" % d["value"], d["unit"], "react %.4f" % d["phase_ms"]["reaction"], "diff %.4f" % d["phase_ms"]["diffusion_and_record"])
        except Exception as e:
            print(c, tag, "ERR", open(f).read()[-300:])
PY
