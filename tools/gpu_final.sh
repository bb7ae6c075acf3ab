#!/bin/bash
# Round-end evidence: full GPU suite, bench (both arms), perf tables, launch
# list, per-kernel instruction census, ncu --set full captures.
set -x
OUT=gpurun_out/final
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python tools/perf.py --reps 20 > $OUT/perf.txt 2>&1
timeout 600 python tools/perf.py --reps 20 --dist uniform --no-f64 > $OUT/perf_u.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-sweep --no-table --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:'k_map_vec|k_sincos_vec|k_f64' --csv --log-file $OUT/inst.csv \
  python tools/perf.py --reps 1 > /dev/null 2>&1
# full captures go to /tmp (gpurun copies back <= 64 MiB); only the raw CSV
# pages and the per-line census come back
REPS=/tmp/final_reps; mkdir -p $REPS
for f in logf log2f log10f log1pf sinf cosf tanf asinf acosf atanf sinhf tanhf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map_vec -s 3 -c 1 \
      -o $REPS/prof_$f python tools/perf.py --fn $f --reps 1 --no-f64 > /dev/null 2>&1
  ncu -i $REPS/prof_$f.ncu-rep --page raw --csv > $OUT/ncu_full_$f.csv 2>/dev/null
  python tools/ncu_lines.py $REPS/prof_$f.ncu-rep 268435456 --top 40 > $OUT/ncu_lines_$f.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_f64 -s 3 -c 1 \
    -o $REPS/prof_exp2d python tools/perf.py --fn f64 --reps 1 > /dev/null 2>&1
ncu -i $REPS/prof_exp2d.ncu-rep --page raw --csv > $OUT/ncu_full_exp2d.csv 2>/dev/null
ls -la $OUT
