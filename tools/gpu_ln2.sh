#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2 or c3" 2>&1 | grep -E "passed|failed|Error"
for v in 1 2; do
  timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_ln2.json 2>/dev/null
  python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_ln2.json"))
c = d["config"]
print("FPS %.1f" % d["value"], {k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()}, "slow", c["slow_pixels_mid"], c["slow_pixel_reasons_per_sweep"])
PY
done
