#!/bin/bash
# round-2 first GPU pass: binary64 hard-set screen, full gpu test suite, bench
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
timeout 900 python tools/hard_cases_f64.py --out tests/golden/hardcases_f64 > $O/hard64.log 2>&1
cp -r tests/golden/hardcases_f64 $O/ 2>/dev/null
timeout 3000 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
tail -c 600 $O/bench.json
