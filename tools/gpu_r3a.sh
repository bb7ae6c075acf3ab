#!/bin/bash
# tanf column-split table variant (sp): exhaustive parity + A/B
OUT=gpurun_out/r3a; mkdir -p $OUT
CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_sp.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_f32.py -k "tanf" > $OUT/pytest_sp.txt 2>&1; echo "rc=$?" >> $OUT/pytest_sp.txt
timeout 900 python tools/ab_interleave.py --fn tanf sinf --rounds 9 base sp > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn tanf --rounds 7 --dist uniform base sp > $OUT/ab_uniform.txt 2>&1
