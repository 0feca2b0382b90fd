#!/bin/bash
# Compare ORd launch-shape variants on C2 (latency regime) and C3 (throughput regime).
# usage: tools/bench_variants.sh "0 1 2" [c3_steps]
VARS=${1:-"0 1 2"}
C3S=${2:-200}
mkdir -p gpurun_out
for v in $VARS; do
  CWG_ORD_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_v$v.log 2>&1; echo "c2 v$v rc=$?"
  CWG_ORD_VARIANT=$v timeout 300 python bench.py --config c3 --steps $C3S --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_v$v.log 2>&1; echo "c3 v$v rc=$?"
done
python - "$VARS" <<'PY'
import json, sys
for v in sys.argv[1].split():
    for c in ("c2", "c3"):
        f = f"gpurun_out/bench_{c}_v{v}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(c, "v" + v, "%.3e" % d["value"], "ms/step %.4f" % d["ms_per_step"], "react %.4f" % d["phase_ms"]["reaction"],
                  "diff %.4f" % d["phase_ms"]["diffusion_and_record"], "fp64frac %.3f" % d["roofline"]["frac"],
                  "meank %.2f" % d["mean_k"], "e2e", d.get("e2e", {}).get("value"), "clk", d["clocks"]["sm_mhz"])
        except Exception as e:
            print(c, v, "ERR", e, open(f).read()[-400:])
PY
