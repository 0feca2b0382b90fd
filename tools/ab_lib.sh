#!/bin/bash
# A/B: default libcwgpu.so vs an alternate build (CWG_LIB_PATH) on C2 and C3.
ALT=$1; C3S=${2:-200}
for tag in base alt; do
  if [ $tag = alt ]; then export CWG_LIB_PATH=$ALT; else unset CWG_LIB_PATH; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_c2_$tag.log 2>&1; echo "c2 $tag rc=$?"
  timeout 300 python bench.py --config c3 --steps $C3S --no-cpu-baseline --no-e2e > gpurun_out/ab_c3_$tag.log 2>&1; echo "c3 $tag rc=$?"
done
python - <<'PY'
import json
for c in ("c2", "c3"):
    for tag in ("base", "alt"):
        f = f"gpurun_out/ab_{c}_{tag}.log"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(c, tag, "%.3e" % d["value"], "react %.4f" % d["phase_ms"]["reaction"], "diff %.4f" % d["phase_ms"]["diffusion_and_record"], "fp64frac %.3f" % d["roofline"]["frac"])
        except Exception as e:
            print(c, tag, "ERR", open(f).read()[-300:])
PY
