#!/bin/bash
# r2x: full gpu suite + smoke on the product; log-family conversion variants
OUT=gpurun_out/r2x; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_f32.py \
    -k "(test_map_kernels_exhaustive_vs_golden or test_element_kernels_exhaustive_vs_golden or test_exhaustive_sweep_vs_golden) and (logf or log2f or log10f or log1pf)" > $OUT/pytest_$v.txt 2>&1; echo "rc=$?" >> $OUT/pytest_$v.txt
done
timeout 900 python tools/ab_interleave.py --fn logf log2f log10f log1pf --rounds 7 base "$@" > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn logf log1pf --rounds 5 --dist uniform base "$@" > $OUT/ab_uniform.txt 2>&1
timeout 600 python tools/perf.py --reps 9 > $OUT/perf.txt 2>&1
