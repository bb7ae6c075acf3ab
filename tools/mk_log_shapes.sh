#!/bin/bash
# Developer: variants of SRC (a csrc copy) with one (vw, nv, minb) shape forced on
# the log-family map kernels: bash tools/mk_log_shapes.sh SRC PREFIX "4:2:3 8:1:3 ..."
SRC=$1; PFX=$2
for s in $3; do
  IFS=: read vw nv mb <<< "$s"
  d=/tmp/var/$PFX$vw$nv$mb; rm -rf $d; cp -r $SRC $d
  python - "$d/crvec_kernels.cuh" $vw $nv $mb <<'PY'
import re, sys
p, vw, nv, mb = sys.argv[1:]
s = open(p).read()
for fn in ("FnLog1p", "FnLog", "FnLog10", "FnLog2"):
    s = re.sub(r"template <> struct KernelShape<%s> \{[^\n]*\n" % fn, "", s)
anchor = "template <> struct KernelShape<FnExp2>"
add = "".join("template <> struct KernelShape<%s> { static constexpr int vw = %s, nv = %s, minb = %s; };\n" % (fn, vw, nv, mb)
              for fn in ("FnLog1p", "FnLog", "FnLog10", "FnLog2"))
s = s.replace(anchor, add + anchor)
open(p, "w").write(s)
PY
done
for s in $3; do
  IFS=: read vw nv mb <<< "$s"
  python -m paper_2605_15547_b200.build --variant $PFX$vw$nv$mb /tmp/var/$PFX$vw$nv$mb > /tmp/var/$PFX$vw$nv$mb.log 2>&1 &
done
wait
for s in $3; do IFS=: read vw nv mb <<< "$s"; tail -n 1 /tmp/var/$PFX$vw$nv$mb.log; done
rm -rf paper_2605_15547_b200/variants/_build_*
