#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_reference_parity.py -q -s -k c5 > gpurun_out/r2/refparity_c5c.log 2>&1
grep -E "^C[0-9]|^  [a-z]|passed|failed" gpurun_out/r2/refparity_c5c.log | head -20
timeout 900 python bench.py --train-only --no-cpu-baseline > gpurun_out/r2/bench_train.json 2>gpurun_out/r2/bench_train.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_train.json"))["train"]
print("train it/s %.1f e2e %.1f" % (d["value"], d["e2e"]["value"]), {k: round(v, 4) for k, v in d["stage_ms_one_step"].items()})
PY
