#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_train.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2" 2>&1 | grep -E "passed|failed"
for v in 2 2; do
  timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_k1.json 2>gpurun_out/r2/bench_k1.err
  python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_k1.json"))
print("FPS %.1f" % d["value"], {k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()})
print({k: round(v["frac"], 3) for k, v in d["kernels"].items()})
PY
done
VIEWS=1 timeout 900 python tools/diag_c5_backward.py 2>&1 | tail -8
