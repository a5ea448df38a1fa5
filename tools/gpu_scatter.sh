#!/bin/bash
# Tile-major scatter: parity (forward / backward / reference / training) and the render + train legs.
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py tests/test_gpu_train.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_forward.py -q -s -k binning_modes 2>&1 | grep -E "pairs|passed|failed"
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2" 2>&1 | grep -E "passed|failed|Error|assert"
timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_sc.json 2>gpurun_out/r2/bench_sc.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_sc.json"))
print("render FPS %.1f" % d["value"], {k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()})
PY
timeout 900 python bench.py --train-only --no-cpu-baseline --no-dropin > gpurun_out/r2/bench_tr.json 2>/dev/null
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2/bench_tr.json"))["train"]
print("train", round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: round(v,3) for k,v in d["stage_ms_one_step"].items()})
PY
