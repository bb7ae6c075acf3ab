#!/bin/bash
# tanh / asin / acos shapes (w823, w442): exhaustive map-kernel parity + A/B
OUT=gpurun_out/r3d; mkdir -p $OUT
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "test_map_kernels_exhaustive_vs_golden and (tanhf or asinf or acosf)" > $OUT/pytest_$v.txt 2>&1; echo "rc=$?" >> $OUT/pytest_$v.txt
done
timeout 900 python tools/ab_interleave.py --fn tanhf asinf acosf --rounds 9 base "$@" > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn tanhf asinf acosf --rounds 7 --dist uniform base "$@" > $OUT/ab_uniform.txt 2>&1
