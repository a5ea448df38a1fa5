#!/bin/bash
# Quick render check on the GPU box: forward/backward parity tests + render bench (no train/e2e/CPU legs).
timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-train --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("FPS", round(d["value"], 1), "ms/frame", round(d["ms_per_frame"], 4))
print({k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()})
c = d["config"]
print("E_kernel/frame %.1fM  E %.1fM  B %.1fM  slow %d" % (c["kernel_evals_per_frame"] / 1e6, c["evals_per_frame"] / 1e6,
      c["blends_per_frame"] / 1e6, c["slow_pixels_mid"]))
PY
