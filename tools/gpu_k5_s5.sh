#!/bin/bash
# A/B: K5 early colour loads (default) vs late (RGS_K5=4); parity of the default.
mkdir -p gpurun_out/s5
timeout 400 python -m pytest tests/test_gpu_forward.py -m gpu -x -q > gpurun_out/s5/tests.log 2>&1; echo rc=$? >> gpurun_out/s5/tests.log
for v in 2 4 2 4; do
  RGS_K5=$v timeout 300 python bench.py --no-train --no-c4 --no-c5 --no-cpu-baseline --no-dropin --no-e2e > gpurun_out/s5/bench_$v.json 2>> gpurun_out/s5/bench.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5/bench_$v.json').read().strip().splitlines()[-1])
print('K5=$v', round(d['value'],1), d['stages']['blend_fp32_k5']['ms_per_frame'])" >> gpurun_out/s5/ab.txt
done
cat gpurun_out/s5/ab.txt
