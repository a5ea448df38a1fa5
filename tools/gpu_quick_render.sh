#!/bin/bash
mkdir -p gpurun_out/r2
timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_q.json 2>gpurun_out/r2/bench_q.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_q.json"))
print("render FPS %.1f" % d["value"])
print(json.dumps(d["binning"], indent=1))
PY
tail -3 gpurun_out/r2/bench_q.err
