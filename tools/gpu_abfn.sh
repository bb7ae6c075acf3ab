#!/bin/bash
# A/B of variant builds on a function subset, config + uniform inputs:
#   bash tools/gpu_abfn.sh TAG "fn1 fn2 ..." base var1 var2 ...   (base = the product libcrvec.so)
TAG=$1; FNS=$2; shift 2
OUT=gpurun_out/abfn_$TAG; mkdir -p $OUT
for rep in 1 2; do
for v in "$@"; do
  lib=paper_2605_15547_b200/variants/libcrvec_$v.so; [ "$v" = base ] && lib=paper_2605_15547_b200/libcrvec.so
  CRVEC_LIB=$lib timeout 300 python tools/perf.py --no-f64 --reps 20 --fn $FNS > $OUT/${v}_$rep.txt 2>&1
  CRVEC_LIB=$lib timeout 300 python tools/perf.py --no-f64 --reps 20 --dist uniform --fn $FNS > $OUT/${v}_u_$rep.txt 2>&1
done; done
python - "$OUT" "$@" <<'PY' | tee $OUT/table.txt
import json, sys, os
out, vs = sys.argv[1], sys.argv[2:]
for suf, title in (("", "config"), ("_u", "uniform")):
    tab = {}
    for v in vs:
        for rep in (1, 2):
            p = os.path.join(out, f"{v}{suf}_{rep}.txt")
            if not os.path.exists(p): continue
            for l in open(p):
                if l.startswith("{"):
                    d = json.loads(l); tab.setdefault(d["fn"], {}).setdefault(v, []).append(d["gelem_s"])
    print(f"-- {title} (Gelem/s, best of 2 runs)\nfn       " + " ".join(f"{v:>8s}" for v in vs))
    for fn, r in tab.items():
        print(f"{fn:8s} " + " ".join(f"{max(r.get(v, [0])):8.1f}" for v in vs))
PY
