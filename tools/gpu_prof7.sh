#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/perf.py > gpurun_out/perf7.txt 2>&1
timeout 300 python tools/perf.py --dist uniform --no-f64 --fn sinf cosf tanf sincosf logf log1pf > gpurun_out/perf7u.txt 2>&1
for f in logf expf sinf asinf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map_vec -s 3 -c 1 -o gpurun_out/prof7_$f python tools/perf.py --fn $f --reps 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_f64 -s 3 -c 1 -o gpurun_out/prof7_exp2d python tools/perf.py --reps 1 --fn f64 > /dev/null 2>&1
