#!/bin/bash
# K5 A/B: parity tests with the new kernel, then the render bench with RGS_K5=1 (round-1 kernel) and default.
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2 or c3" 2>&1 | grep -E "^C|passed|failed"
for v in 1 2 1 2; do
  RGS_K5=$v timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_k5_$v.json 2>gpurun_out/r2/bench_k5_$v.err
  python - $v <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2/bench_k5_{sys.argv[1]}.json"))
c = d["config"]
print("K5 variant", sys.argv[1], "FPS %.1f" % d["value"], "K5 serial ms %.4f" % d["stages"]["blend_fp32_k5"]["ms_per_frame"],
      "frac_serial %.3f live %.3f" % (d["roofline"]["frac_serialised"], d["roofline"]["frac"]),
      "slow %d" % c["slow_pixels_mid"], "reasons", c["slow_pixel_reasons_per_sweep"])
PY
done
