#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -x -q -s -k "c1 or c2" 2>&1 | grep -E "passed|failed|Error"
bash tools/gpu_k1ab.sh
