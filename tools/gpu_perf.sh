#!/bin/bash
# usage: bash tools/gpu_perf.sh TAG  -> gpurun_out/perf_TAG.txt, perf_TAG_u.txt
mkdir -p gpurun_out
timeout 600 python tools/perf.py > gpurun_out/perf_$1.txt 2>&1
timeout 300 python tools/perf.py --dist uniform --no-f64 --fn sinf cosf tanf sincosf logf log1pf asinf expm1f tanhf > gpurun_out/perf_$1_u.txt 2>&1
