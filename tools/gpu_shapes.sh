#!/bin/bash
# bash tools/gpu_shapes.sh TAG var...  -> per-variant perf tables (config dist, all fns)
TAG=$1; shift
OUT=gpurun_out/shapes_$TAG; mkdir -p $OUT
for v in "$@"; do
  CRVEC_LIB=paper_2605_15547_b200/variants/libcrvec_$v.so timeout 400 python tools/perf.py --no-f64 > $OUT/$v.txt 2>&1
done
python - "$OUT" "$@" <<'PY'
import json, sys, os
out, vs = sys.argv[1], sys.argv[2:]
tab = {}
for v in vs:
    for l in open(os.path.join(out, v + ".txt")):
        if l.startswith("{"):
            d = json.loads(l); tab.setdefault(d["fn"], {})[v] = d["gelem_s"]
print("fn       " + " ".join(f"{v:>7s}" for v in vs))
for fn, r in tab.items():
    print(f"{fn:8s} " + " ".join(f"{r.get(v, 0):7.1f}" for v in vs))
PY
