#!/bin/bash
# r2z: acos fourth-column variant (a1), tanh conversion variant (t1): exhaustive parity + A/B
OUT=gpurun_out/r2z; mkdir -p $OUT
CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_a1.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "acosf" > $OUT/pytest_a1.txt 2>&1; echo "rc=$?" >> $OUT/pytest_a1.txt
CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_t1.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "tanhf" > $OUT/pytest_t1.txt 2>&1; echo "rc=$?" >> $OUT/pytest_t1.txt
timeout 900 python tools/ab_interleave.py --fn acosf tanhf --rounds 9 base a1 t1 > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn acosf tanhf --rounds 7 --dist uniform base a1 t1 > $OUT/ab_uniform.txt 2>&1
