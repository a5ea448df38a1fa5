#!/bin/bash
# Turns a milestone's gpurun_out/r2 captures into the tracked summaries under profiles/ (run here).
set -e
R=${1:-r2}
G=gpurun_out/$R
P=profiles
{ echo "# ncu launch list of the C2 render sweep ($R; cold-cache, serialised: compare shares)"; echo
  python tools/launch_summary.py $G/launches_render.csv; } > $P/ncu_launches_render_$R.md
{ echo "# ncu launch list of C3 training steps ($R; cold-cache, serialised: compare shares)"; echo
  python tools/launch_summary.py $G/launches_train.csv; } > $P/ncu_launches_train_$R.md
cp $G/launches_render.csv $P/ncu_launches_render_$R.csv
cp $G/launches_train.csv $P/ncu_launches_train_$R.csv
python tools/ncu_summary.py $G/prof_render.ncu-rep > $P/ncu_full_render_$R.md
python tools/ncu_summary.py $G/prof_train.ncu-rep > $P/ncu_full_train_$R.md
python tools/ncu_stalls.py $G/prof_render.ncu-rep 'k_blend_fp32|k_preprocess|k_radix|k_duplicate|k_slice_cache' > $P/ncu_stalls_render_$R.md
python tools/ncu_stalls.py $G/prof_train.ncu-rep 'k_backward_fp32|k_gaussian_backward|k_color_backward|k_ssim|k_image_grad|k_adam|k_tile_scatter|k_chunk_tile_counts|k_tile_offsets' > $P/ncu_stalls_train_$R.md
cp $G/bench_full.json $P/bench_${R}_full.json
ls -la $P | grep $R
