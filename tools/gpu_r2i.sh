#!/bin/bash
timeout 300 python tools/diag_repro.py 2>&1 | tail -12
bash tools/gpu_radix_ab.sh
