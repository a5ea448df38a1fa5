#!/bin/bash
# End-of-milestone pass on the GPU box (run under gpurun): GPU tests, the default bench line,
# launch lists of the render sweep and the training step, and ncu --set full captures of the
# hot kernels.  Outputs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 100 --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile-only --warmup 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv \
    --log-file gpurun_out/launches_train.csv python bench.py --train-only --train-steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_blend_fp32|k_preprocess|k_radix_onesweep|k_duplicate' -s 40 -c 4 \
    -o gpurun_out/prof_full python bench.py --profile-only --warmup 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_backward_fp32|k_gaussian_backward|k_color_backward|k_adam_step|k_ssim_fields|k_image_grad' -s 8 -c 6 \
    -o gpurun_out/prof_train python bench.py --train-only --train-steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_train.log 2>&1
tail -3 gpurun_out/ncu_full.log gpurun_out/ncu_train.log
ls -la gpurun_out
