#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_backward.py tests/test_gpu_reference_suite.py -q -s 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|reproducible:" | tail -30
timeout 900 python bench.py --train-only --no-cpu-baseline > gpurun_out/r2/bench_t2.json 2>gpurun_out/r2/bench_t2.err
tail -2 gpurun_out/r2/bench_t2.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_t2.json"))["train"]
print("train it/s %.1f e2e %.1f" % (d["value"], d["e2e"]["value"]))
print("dropin", d["dropin"])
PY
