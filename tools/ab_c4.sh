#!/bin/bash
# A/B on the headline config: reaction / diffusion ms per step for libraries
# given as name=path pairs (CWG_LIB_PATH), N steps each, alternated twice.
# usage: tools/ab_c4.sh "base=alt/libcwgpu_base.so new=paper_2011_04747_b200/libcwgpu.so" [steps] [config]
PAIRS=$1; STEPS=${2:-300}; CFG=${3:-c4}
mkdir -p gpurun_out
for rep in 1 2; do
  for pr in $PAIRS; do
    tag=${pr%%=*}; lib=${pr#*=}
    CWG_LIB_PATH=$lib timeout 600 python bench.py --config $CFG --steps $STEPS --warmup 5 --no-cpu-baseline --no-e2e \
      > gpurun_out/ab_${CFG}_${tag}_$rep.log 2>&1; echo "$CFG $tag rep$rep rc=$?"
  done
done
python - "$PAIRS" $CFG <<'PY'
import json, sys
cfg = sys.argv[2]
for pr in sys.argv[1].split():
    tag = pr.split("=")[0]
    for rep in (1, 2):
        f = f"gpurun_out/ab_{cfg}_{tag}_{rep}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(cfg, tag, rep, "%.4e" % d["value"], "ms/step %.4f" % d["ms_per_step"], "react %.4f" % d["phase_ms"]["reaction"],
                  "diff %.4f" % d["phase_ms"]["diffusion_and_record"], "fp64frac %.3f" % d["roofline"]["frac"],
                  "meank %.3f" % d["mean_k"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
        except Exception as e:
            print(cfg, tag, rep, "ERR", e, open(f).read()[-400:])
PY
