#!/bin/bash
# Iteration check on the GPU box: full GPU suite + per-function perf table.
# usage: bash tools/gpu_iter.sh TAG  -> gpurun_out/it_TAG/{pytest,perf,perf_u}.txt
OUT=gpurun_out/it_$1
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1
tail -3 $OUT/pytest.txt
timeout 600 python tools/perf.py > $OUT/perf.txt 2>&1
timeout 300 python tools/perf.py --dist uniform --no-f64 > $OUT/perf_u.txt 2>&1
tail -23 $OUT/perf.txt
tail -21 $OUT/perf_u.txt
