#!/bin/bash
# r2y: binary64 exp2 round-test bound as one constant (variant f1): f64 gpu tests + A/B
OUT=gpurun_out/r2y; mkdir -p $OUT
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f64.py > $OUT/pytest_f64_$v.txt 2>&1; echo "rc=$?" >> $OUT/pytest_f64_$v.txt
done
timeout 900 python tools/ab_interleave.py --fn f64 --rounds 9 base "$@" > $OUT/ab_f64.txt 2>&1
