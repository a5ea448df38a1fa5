#!/bin/bash
mkdir -p gpurun_out/r2
timeout 2300 python -m pytest tests/test_gpu_sanitizer.py -q -s 2>&1 | grep -E "SUMMARY|passed|failed" | head -10
timeout 900 python -m pytest tests/test_gpu_forward.py -q -x 2>&1 | tail -1
timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_q.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r2/bench_q.json')); print('FPS', d['value'], d['binning']['scatter']['stages_ms_per_frame'])"
