#!/bin/bash
# A/B of K5 variants (RGS_K5=...): render-only bench, K5 serialised ms per C2 frame.  Usage: gpu_k5_ab.sh OUT v1 v2 ...
out=gpurun_out/$1; shift
mkdir -p $out
timeout 400 python -m pytest tests/test_gpu_forward.py -m gpu -x -q > $out/tests.log 2>&1; echo rc=$? >> $out/tests.log
for rep in 1 2; do for v in "$@"; do
  RGS_K5=$v timeout 300 python bench.py --no-train --no-c4 --no-c5 --no-cpu-baseline --no-dropin --no-e2e > $out/bench_$v.json 2>> $out/bench.err
  python -c "
import json;d=json.loads(open('$out/bench_$v.json').read().strip().splitlines()[-1])
print('K5=$v', round(d['value'],1), round(d['stages']['blend_fp32_k5']['ms_per_frame'],4), d['config']['slow_pixels_mid'])" >> $out/ab.txt
done; done
tail -1 $out/tests.log; cat $out/ab.txt
