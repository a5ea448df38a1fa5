#!/bin/bash
# Profiling pass on the GPU box (run under gpurun): ncu full captures of the render and
# training hot kernels and launch lists; outputs in gpurun_out/.
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_blend_fp32|k_preprocess|k_radix_scatter' -s 60 -c 3 \
    -o gpurun_out/prof_render python bench.py --profile-only --warmup 1 > gpurun_out/ncu_render.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_backward_fp32|k_gaussian_backward|k_adam_step|k_ssim_fields|k_image_grad|k_knn' -s 8 -c 6 \
    -o gpurun_out/prof_train python bench.py --train-only --train-steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_train.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 100 --csv \
    --log-file gpurun_out/launches_render.csv python bench.py --profile-only --warmup 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv \
    --log-file gpurun_out/launches_train.csv python bench.py --train-only --train-steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
