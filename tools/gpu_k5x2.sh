#!/bin/bash
mkdir -p gpurun_out/r2
RGS_K5=3 timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -x -q 2>&1 | tail -2
RGS_K5=3 timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2" 2>&1 | grep -E "passed|failed|Error"
for v in 2 3 2 3; do
  RGS_K5=$v timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_x2_$v.json 2>gpurun_out/r2/bench_x2_$v.err
  python - $v <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2/bench_x2_{sys.argv[1]}.json"))
c = d["config"]
print("K5 variant", sys.argv[1], "FPS %.1f" % d["value"], "K5 serial ms %.4f" % d["stages"]["blend_fp32_k5"]["ms_per_frame"],
      "frac_serial %.3f" % d["roofline"]["frac_serialised"], "E_kernel/frame %.1fM" % (c["kernel_evals_per_frame"] / 1e6),
      "slow", c["slow_pixels_mid"])
PY
done
