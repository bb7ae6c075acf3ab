#!/bin/bash
# Developer: build variants with one (NV, MINB) kernel shape forced on every
# binary32 map kernel: bash tools/mk_shape_variants.sh "1:4 2:2 2:3 ..."
for s in $1; do
  nv=${s%:*}; mb=${s#*:}
  d=/tmp/var/s$nv$mb; rm -rf $d; cp -r paper_2605_15547_b200/csrc $d
  python - "$d/crvec_kernels.cuh" $nv $mb <<'PY'
import re, sys
p, nv, mb = sys.argv[1], sys.argv[2], sys.argv[3]
s = open(p).read()
s = re.sub(r"static constexpr int vw = 4, nv = \d+, minb = \d+;", f"static constexpr int vw = 4, nv = {nv}, minb = {mb};", s)
open(p, "w").write(s)
PY
done
for s in $1; do
  nv=${s%:*}; mb=${s#*:}
  python -m paper_2605_15547_b200.build --variant s$nv$mb /tmp/var/s$nv$mb > /tmp/var/s$nv$mb.log 2>&1 &
done
wait
for s in $1; do nv=${s%:*}; mb=${s#*:}; tail -n 1 /tmp/var/s$nv$mb.log; done
rm -rf paper_2605_15547_b200/variants/_build_*
