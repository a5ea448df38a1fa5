#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s -k "reproducible" 2>&1 | tail -30
