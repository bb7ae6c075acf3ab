#!/bin/bash
# L2 bulk prefetch for the issue-bound kernels (variant pf): parity + A/B
OUT=gpurun_out/r3b; mkdir -p $OUT
CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_pf.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "test_map_kernels_exhaustive_vs_golden and (sinhf or atanf or tanhf or asinf or acosf or sinf or cosf or tanf)" > $OUT/pytest_pf.txt 2>&1; echo "rc=$?" >> $OUT/pytest_pf.txt
timeout 900 python tools/ab_interleave.py --fn sinhf atanf tanhf asinf acosf sinf tanf --rounds 7 base pf > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn sinhf atanf tanhf asinf acosf sinf tanf --rounds 5 --dist uniform base pf > $OUT/ab_uniform.txt 2>&1
