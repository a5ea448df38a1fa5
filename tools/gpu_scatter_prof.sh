#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_|k_chunk_tile' -s 20 -c 4 \
    -o gpurun_out/r2/prof_scatter2 python bench.py --profile-only --warmup 1 > gpurun_out/r2/ncu_sc.log 2>&1
tail -2 gpurun_out/r2/ncu_sc.log
