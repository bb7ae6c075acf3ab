#!/bin/bash
mkdir -p gpurun_out/hardcases
bash tools/gpu_perf.sh v11
CRVEC_HARDCASE_OUT=gpurun_out/hardcases timeout 900 python tools/hard_cases.py > gpurun_out/hardcases.log 2>&1
timeout 600 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err
