#!/bin/bash
# round-2 GPU pass: binary64 hard-set screen, full gpu test suite, bench (both arms), ncu launch list
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
timeout 900 python tools/hard_cases_f64.py --out tests/golden/hardcases_f64 > $O/hard64.log 2>&1
cp -r tests/golden/hardcases_f64 $O/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
tail -c 1500 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
tail -c 600 $O/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-table > $O/ncu_bench.log 2>&1
echo ncu rc $?
