#!/bin/bash
# round-2 evidence pass: gpu tests, smoke, bench (both arms), ncu launch list, ncu --set full of the log-family kernels
O=gpurun_out/r2m; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-table > $O/ncu_bench.log 2>&1
for fn in log1pf logf; do
  k=$([ $fn = log1pf ] && echo FnLog1p || echo "FnLogBILi0")
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$k -c 1 -o $O/ncu_full_$fn python tools/perf.py --fn $fn --reps 1 --no-f64 > $O/ncu_$fn.log 2>&1
  ncu -i $O/ncu_full_$fn.ncu-rep --page raw --csv > $O/ncu_full_$fn.csv 2>/dev/null
done
ls -la $O
