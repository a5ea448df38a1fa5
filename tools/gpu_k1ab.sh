#!/bin/bash
mkdir -p gpurun_out/r2
for v in a b; do
  timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_k1_$v.json 2>/dev/null
  python - $v <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2/bench_k1_{sys.argv[1]}.json"))
print("FPS %.1f" % d["value"], {k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()})
PY
done
