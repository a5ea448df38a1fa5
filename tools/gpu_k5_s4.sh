#!/bin/bash
# K5 instruction cuts: parity (forward, backward, reference build), render bench, one ncu capture of K5.
mkdir -p gpurun_out/s4
timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py tests/test_gpu_reference_parity.py -m gpu -x -q > gpurun_out/s4/tests.log 2>&1; echo rc=$? >> gpurun_out/s4/tests.log
timeout 300 python bench.py --no-train --no-c4 --no-c5 --no-cpu-baseline --no-dropin > gpurun_out/s4/bench.json 2> gpurun_out/s4/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_blend_fp32' -s 40 -c 2 \
    -o gpurun_out/s4/prof_k5 python bench.py --profile-only --warmup 1 > gpurun_out/s4/ncu_k5.log 2>&1
tail -3 gpurun_out/s4/ncu_k5.log
