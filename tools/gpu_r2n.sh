#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_train.py -x -q -s -k "trajectory" 2>&1 | grep -E "trajectory|passed|failed|Error|assert" | head
timeout 900 python bench.py --train-only --no-cpu-baseline --no-dropin > gpurun_out/r2/bench_t3.json 2>gpurun_out/r2/bench_t3.err
tail -2 gpurun_out/r2/bench_t3.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_t3.json"))["train"]
print("train it/s %.1f repro %.1f f64 %.1f" % (d["value"], d["reproducible"]["value"], d["f64_scene"]["value"]))
PY
