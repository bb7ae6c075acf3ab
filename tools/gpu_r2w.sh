#!/bin/bash
# r2w: kernel-shape re-tune after the div/sqrt series change (variants sA, sB)
OUT=gpurun_out/r2w; mkdir -p $OUT
timeout 1200 python tools/ab_interleave.py --fn tanf tanhf atanf asinf acosf sinf cosf --rounds 7 base "$@" > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn tanf tanhf atanf asinf acosf sinf cosf --rounds 5 --dist uniform base "$@" > $OUT/ab_uniform.txt 2>&1
