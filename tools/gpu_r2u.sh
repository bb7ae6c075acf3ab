#!/bin/bash
# Round 2 (r2u): MUFU seed probe, exhaustive parity of the variant builds on
# the functions they change, interleaved A/B against the product library.
#   bash tools/gpu_r2u.sh TAG "fn ..." var ...
TAG=$1; FNS=$2; shift 2
OUT=gpurun_out/r2u_$TAG; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_probe.cu -o /tmp/mufu_probe && /tmp/mufu_probe > $OUT/mufu_probe.txt 2>&1
K=$(echo $FNS | sed 's/ / or /g')
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 1500 python -m pytest -q -x -m gpu \
    tests/test_gpu_f32.py -k "(test_map_kernels_exhaustive_vs_golden or test_element_kernels_exhaustive_vs_golden or test_exhaustive_sweep_vs_golden) and ($K)" \
    > $OUT/pytest_$v.txt 2>&1; echo "rc=$?" >> $OUT/pytest_$v.txt
done
timeout 1200 python tools/ab_interleave.py --fn $FNS --rounds 7 base "$@" > $OUT/ab_config.txt 2>&1
timeout 900 python tools/ab_interleave.py --fn $FNS --rounds 5 --dist uniform base "$@" > $OUT/ab_uniform.txt 2>&1
tail -30 $OUT/ab_config.txt
