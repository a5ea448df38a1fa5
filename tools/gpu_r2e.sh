#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -s 2>&1 | grep -E "rank|passed|failed|Error|error" | head -20
timeout 900 python -m pytest tests/test_gpu_train.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_reference_parity.py -q -s -k c5 > gpurun_out/r2/refparity_c5b.log 2>&1
grep -E "^C[0-9]|^  [a-z]|passed|failed" gpurun_out/r2/refparity_c5b.log | head -40
