#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --train-only --no-cpu-baseline > gpurun_out/r2/bench_tr.json 2>/dev/null
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_tr.json"))["train"]
print("train", round(d["value"],1), "e2e", round(d["e2e"]["value"],1))
print(json.dumps(d.get("dropin"), indent=1))
PY
