#!/bin/bash
# K6 / adam / K5 source-level captures (run under gpurun).
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_backward_fp32|k_adam_step' -s 2 -c 2 \
    -o gpurun_out/prof_k6 python bench.py --train-only --train-steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_k6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_blend_fp32' -s 20 -c 1 \
    -o gpurun_out/prof_k5 python bench.py --profile-only --warmup 1 > gpurun_out/ncu_k5.log 2>&1
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -k "adam" 2>&1 | tail -3
timeout 600 python bench.py --train-only --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/train_adam.json
ls gpurun_out
