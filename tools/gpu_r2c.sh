#!/bin/bash
mkdir -p gpurun_out/r2
./tools/probes/pipe_probe
timeout 1500 python -m pytest tests/test_gpu_reference_parity.py -q -s -k c5 > gpurun_out/r2/refparity_c5.log 2>&1
grep -E "^C[0-9]|^  [a-z]|passed|failed" gpurun_out/r2/refparity_c5.log | head -80
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -q -s -k initcheck 2>&1 | tail -3
cp gpurun_out/sanitizer_*.log gpurun_out/r2/ 2>/dev/null
