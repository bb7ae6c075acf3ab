#!/bin/bash
# first GPU round: environment, tests, bench, launch list, one full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_f32.py -q -m gpu -k "not sweep and not accurate_path" -x 2>&1 | tail -40 > gpurun_out/pytest_par.txt
timeout 600 python -m pytest tests/test_gpu_f32.py -q -m gpu -k "sweep and (logf or log2f or log10f or log1pf or expf or exp2f or sinf)" 2>&1 | tail -40 > gpurun_out/pytest_sweep.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_vec -s 4 -c 1 -o gpurun_out/prof_logf python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
