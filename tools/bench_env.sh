#!/bin/bash
# A/B an environment setting on C2 and C3.
# usage: tools/bench_env.sh VAR "v1 v2 ..." [c3_steps]
VAR=$1
VALS=${2:-"1 4"}
C3S=${3:-200}
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_${VAR}_$v.log 2>&1; echo "c2 $VAR=$v rc=$?"
  env $VAR=$v timeout 300 python bench.py --config c3 --steps $C3S --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_${VAR}_$v.log 2>&1; echo "c3 $VAR=$v rc=$?"
done
python - "$VAR" "$VALS" <<'PY'
import json, sys
var = sys.argv[1]
for v in sys.argv[2].split():
    for c in ("c2", "c3"):
        f = f"gpurun_out/bench_{c}_{var}_{v}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(c, var + "=" + v, "%.3e" % d["value"], "ms/step %.4f" % d["ms_per_step"], "react %.4f" % d["phase_ms"]["reaction"],
                  "diff %.4f" % d["phase_ms"]["diffusion_and_record"], "fp64frac %.3f" % d["roofline"]["frac"],
                  "launches", d.get("gpu_launches"), "e2e", d.get("e2e", {}).get("value"), "clk", d["clocks"]["sm_mhz"])
        except Exception as e:
            print(c, v, "ERR", e, open(f).read()[-400:])
PY
