#!/bin/bash
bash tools/gpu_perf.sh v15
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -6 > gpurun_out/pytest15.txt
