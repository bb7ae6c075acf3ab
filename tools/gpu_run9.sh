#!/bin/bash
mkdir -p gpurun_out/hardcases
bash tools/gpu_perf.sh v9
CRVEC_HARDCASE_OUT=gpurun_out/hardcases timeout 900 python tools/hard_cases.py > gpurun_out/hardcases.log 2>&1
timeout 900 python -m pytest tests/test_gpu_f32.py -q -m gpu -k "tanh or random" 2>&1 | tail -5 > gpurun_out/pytest9.txt
