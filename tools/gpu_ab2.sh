#!/bin/bash
# A/B of variant builds over all functions, config + uniform inputs, reps 20:
# bash tools/gpu_ab2.sh TAG var...  -> table
TAG=$1; shift
OUT=gpurun_out/ab2_$TAG; mkdir -p $OUT
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 300 python tools/perf.py --no-f64 --reps 20 > $OUT/$v.txt 2>&1
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 300 python tools/perf.py --no-f64 --reps 20 --dist uniform --fn logf log2f log10f log1pf sinf cosf tanf sincosf > $OUT/${v}_u.txt 2>&1
done
python - "$OUT" "$@" <<'PY'
import json, sys, os
out, vs = sys.argv[1], sys.argv[2:]
for suf, title in (("", "config"), ("_u", "uniform")):
    tab = {}
    for v in vs:
        for l in open(os.path.join(out, v + suf + ".txt")):
            if l.startswith("{"):
                d = json.loads(l); tab.setdefault(d["fn"], {})[v] = d["gelem_s"]
    print(f"-- {title}\nfn       " + " ".join(f"{v:>7s}" for v in vs))
    for fn, r in tab.items():
        print(f"{fn:8s} " + " ".join(f"{r.get(v, 0):7.1f}" for v in vs))
PY
