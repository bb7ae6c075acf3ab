#!/bin/bash
bash tools/gpu_perf.sh v16
timeout 1200 python -m pytest tests/test_gpu_f64.py tests/test_gpu_f32.py -q -m gpu -k "f64 or exp or log or tanh or sweep" 2>&1 | tail -4 > gpurun_out/pytest16.txt
