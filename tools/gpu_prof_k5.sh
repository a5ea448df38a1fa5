#!/bin/bash
mkdir -p gpurun_out/r2
VIEWS=2 timeout 900 python tools/diag_c5_backward.py 2>&1 | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_blend_fp32' -s 40 -c 3 \
    -o gpurun_out/r2/prof_k5v2 python bench.py --profile-only --warmup 1 > gpurun_out/r2/ncu_k5.log 2>&1
tail -3 gpurun_out/r2/ncu_k5.log
