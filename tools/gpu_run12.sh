#!/bin/bash
mkdir -p gpurun_out/hardcases
CRVEC_HARDCASE_OUT=gpurun_out/hardcases timeout 600 python tools/hard_cases.py exp2f log2f > gpurun_out/hardcases2.log 2>&1
timeout 2000 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest12.txt
timeout 300 python tools/perf.py --fn sinf cosf tanf sincosf --no-f64 > gpurun_out/perf12.txt 2>&1
