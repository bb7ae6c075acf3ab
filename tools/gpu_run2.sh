#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/perf.py > gpurun_out/perf2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_f32.py -q -m gpu -x -k "random or config or sizes or scalar or sincos" 2>&1 | tail -15 > gpurun_out/pytest2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_vec -s 3 -c 1 -o gpurun_out/prof_logf2 python tools/perf.py --fn logf --reps 1 > /dev/null 2>&1
