#!/bin/bash
# A/B perf of variant builds: bash tools/gpu_ab.sh TAG "fn ..." var1 var2 ...
TAG=$1; FNS=$2; shift 2
OUT=gpurun_out/ab_$TAG; mkdir -p $OUT
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 300 python tools/perf.py --no-f64 --fn $FNS > $OUT/$v.txt 2>&1
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 300 python tools/perf.py --no-f64 --dist uniform --fn $FNS > $OUT/${v}_u.txt 2>&1
done
for v in "$@"; do echo "== $v config"; grep -A30 "^fn " $OUT/$v.txt | tail -n +2; echo "== $v uniform"; grep -A30 "^fn " $OUT/${v}_u.txt | tail -n +2; done
