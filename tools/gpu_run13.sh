#!/bin/bash
bash tools/gpu_perf.sh v13
timeout 900 python -m pytest tests/test_gpu_f32.py -q -m gpu -k "trig or sincos or sweep or sizes" 2>&1 | tail -4 > gpurun_out/pytest13.txt
