#!/bin/bash
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_reference_parity.py -q -s 2>&1 | tail -40
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -s 2>&1 | tail -20
cp gpurun_out/sanitizer_*.log gpurun_out/r2/ 2>/dev/null
for f in gpurun_out/r2/sanitizer_*.log; do echo "== $f"; grep -E "SUMMARY|Error|error" $f | head -5; done
