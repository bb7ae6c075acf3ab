#!/bin/bash
# log family column-split (c, L) table (variant ls): exhaustive parity + A/B
OUT=gpurun_out/r3f; mkdir -p $OUT
CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_ls.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "(test_map_kernels_exhaustive_vs_golden or test_element_kernels_exhaustive_vs_golden or test_exhaustive_sweep_vs_golden) and (logf or log2f or log10f or log1pf)" > $OUT/pytest_ls.txt 2>&1; echo "rc=$?" >> $OUT/pytest_ls.txt
timeout 900 python tools/ab_interleave.py --fn logf log2f log10f log1pf --rounds 9 base ls > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn logf log1pf --rounds 7 --dist uniform base ls > $OUT/ab_uniform.txt 2>&1
