#!/bin/bash
# Round-2 first pass: GPU tests + full bench line (training legs at SH degree 3).
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -k "not reference_suite" 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/r2/bench_a.json 2> gpurun_out/r2/bench_a.err; tail -5 gpurun_out/r2/bench_a.err
