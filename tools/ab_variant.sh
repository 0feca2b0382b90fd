#!/bin/bash
# A/B of ORd launch shapes (CWG_ORD_VARIANT) on one library: reaction ms per step, alternated twice.
# usage: tools/ab_variant.sh "1 4" [steps] [config]
VARS=$1; STEPS=${2:-300}; CFG=${3:-c4}
mkdir -p gpurun_out
for rep in 1 2; do
  for v in $VARS; do
    CWG_ORD_VARIANT=$v timeout 600 python bench.py --config $CFG --steps $STEPS --warmup 5 --no-cpu-baseline --no-e2e \
      > gpurun_out/abv_${CFG}_v${v}_$rep.log 2>&1; echo "$CFG v$v rep$rep rc=$?"
  done
done
python - "$VARS" $CFG <<'PY'
import json, sys
cfg = sys.argv[2]
for v in sys.argv[1].split():
    for rep in (1, 2):
        f = f"gpurun_out/abv_{cfg}_v{v}_{rep}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(cfg, "v" + v, rep, "%.4e" % d["value"], "ms/step %.4f" % d["ms_per_step"], "react %.4f" % d["phase_ms"]["reaction"],
                  "diff %.4f" % d["phase_ms"]["diffusion_and_record"], "meank %.3f" % d["mean_k"])
        except Exception as e:
            print(cfg, v, rep, "ERR", e, open(f).read()[-400:])
PY
