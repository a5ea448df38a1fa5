#!/bin/bash
# Round-2 milestone pass: the default bench line, launch lists of the render sweep and of the
# training step, ncu --set full captures of the hot kernels.  Outputs in gpurun_out/$OUT/.
OUT=${1:-r2}
mkdir -p gpurun_out/$OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python bench.py > gpurun_out/$OUT/bench_full.json 2> gpurun_out/$OUT/bench_full.err; tail -2 gpurun_out/$OUT/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 120 --csv \
    --log-file gpurun_out/$OUT/launches_render.csv python bench.py --profile-only --warmup 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv \
    --log-file gpurun_out/$OUT/launches_train.csv python bench.py --train-only --train-steps 3 --warmup 1 --no-cpu-baseline --no-dropin > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_blend_fp32|k_preprocess|k_radix_onesweep|k_duplicate|k_slice_cache' -s 40 -c 6 \
    -o gpurun_out/$OUT/prof_render python bench.py --profile-only --warmup 1 > gpurun_out/$OUT/ncu_render.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_backward_fp32|k_gaussian_backward|k_color_backward|k_adam|k_ssim_fields|k_image_grad|k_tile_scatter|k_chunk_tile_counts|k_tile_offsets' -s 8 -c 11 \
    -o gpurun_out/$OUT/prof_train python bench.py --train-only --train-steps 1 --warmup 1 --no-cpu-baseline --no-dropin > gpurun_out/$OUT/ncu_train.log 2>&1
tail -2 gpurun_out/$OUT/ncu_render.log gpurun_out/$OUT/ncu_train.log
ls -la gpurun_out/$OUT | tail -12
