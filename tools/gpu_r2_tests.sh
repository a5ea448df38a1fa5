#!/bin/bash
mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2/gpu_tests.log 2>&1
tail -3 gpurun_out/r2/gpu_tests.log
grep -E "^C[0-9]|^  [a-z_]+ +above|^rank|^reproducible:|^[0-9]+x[0-9]+:|^order|PASS|FAIL|test cases|SUMMARY|^memcheck|^racecheck|^initcheck|^synccheck" gpurun_out/r2/gpu_tests.log | head -80
cp gpurun_out/sanitizer_*.log gpurun_out/r2/ 2>/dev/null
