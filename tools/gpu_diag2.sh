#!/bin/bash
timeout 1200 python tools/diag_c5_b.py 2>&1 | tail -45
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -s -k "wide_tile or max_image" 2>&1 | grep -E "x[0-9]|passed|failed|Error"
