#!/bin/bash
# tanf kernel shape with the split table (t22: 8:2:2, t14: 8:1:4): A/B
OUT=gpurun_out/r3c; mkdir -p $OUT
timeout 900 python tools/ab_interleave.py --fn tanf --rounds 9 base "$@" > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn tanf --rounds 7 --dist uniform base "$@" > $OUT/ab_uniform.txt 2>&1
