#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_train.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -k "checkpoint or golden or records" 2>&1 | tail -1
RGS_DROPIN_TRACE=1 timeout 900 python bench.py --train-only --no-cpu-baseline > gpurun_out/r2/bench_tr.json 2>gpurun_out/r2/trace.err
grep -E "^(adam|bwd)" gpurun_out/r2/trace.err | tail -12
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_tr.json"))["train"]
print("train", round(d["value"],1), "e2e", round(d["e2e"]["value"],1))
dd = d.get("dropin"); print("dropin", dd["value"], dd["step_ms"], {k: round(v,1) for k,v in dd["step_breakdown_ms"].items()})
PY
