#!/bin/bash
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -1
RGS_RADIX=8 timeout 600 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -1
for v in 16 8 16 8; do
  RGS_RADIX=$v timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_rx_$v.json 2>gpurun_out/r2/bench_rx_$v.err
  python - $v <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2/bench_rx_{sys.argv[1]}.json"))
print("radix", sys.argv[1], "FPS %.1f" % d["value"], {k: round(v["ms_per_frame"], 4) for k, v in d["stages"].items()})
PY
done
