#!/bin/bash
# Round-end evidence: full GPU suite, bench (both arms), launch list, ncu captures, perf table.
set -x
OUT=gpurun_out/final
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python tools/perf.py > $OUT/perf.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-sweep --no-table --no-cpu > /dev/null 2>&1
for f in logf log1pf expf sinf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map_vec -s 3 -c 1 \
      -o $OUT/prof_$f python tools/perf.py --fn $f --reps 1 > /dev/null 2>&1
done
ls -la $OUT
