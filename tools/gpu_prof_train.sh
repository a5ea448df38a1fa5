#!/bin/bash
# ncu --set full of each training kernel (one launch each, after the warm-up step); run under gpurun.
for k in k_backward_fp32 k_gaussian_backward k_color_backward k_adam_plain k_adam_step k_ssim_fields k_image_grad k_backward_fp64 k_blend_fp64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}\$|::${k}\$|${k}<" -s 6 -c 1 \
      -o gpurun_out/prof_${k} python bench.py --train-only --train-steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_${k}.log 2>&1
done
ls gpurun_out/*.ncu-rep
