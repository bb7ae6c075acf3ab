#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/perf.py > gpurun_out/perf4.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_f32.py -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest4.txt
