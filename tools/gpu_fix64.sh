#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py tests/test_gpu_train.py -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -k "c1 or c2 or c3" 2>&1 | tail -1
timeout 600 python bench.py --no-train --no-c4 --no-c5 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r2/bench_q.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r2/bench_q.json')); print('FPS', round(d['value'],1), {k:round(v['ms_per_frame'],4) for k,v in d['stages'].items()})"
timeout 900 python bench.py --train-only --no-cpu-baseline --no-dropin > gpurun_out/r2/bench_tr.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r2/bench_tr.json'))['train']; print('train', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['stage_ms_one_step'].items()})"
