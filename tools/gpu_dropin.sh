#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python bench.py --train-only --no-cpu-baseline --train-steps 5 > gpurun_out/r2/bench_dropin.json 2>gpurun_out/r2/bench_dropin.err
tail -3 gpurun_out/r2/bench_dropin.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_dropin.json"))["train"]
print("train it/s %.1f" % d["value"], "dropin", d["dropin"])
PY
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q 2>&1 | tail -3
