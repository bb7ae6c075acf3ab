#!/bin/bash
# Developer: variants of SRC (a csrc copy) with one (vw, nv, minb) shape forced
# on the KernelShape specialisations whose line matches PATTERN:
#   bash tools/mk_fn_shapes.sh SRC PREFIX 'FnTrig<W>' "4:2:2 8:1:3 ..."
SRC=$1; PFX=$2; PAT=$3
for s in $4; do
  IFS=: read vw nv mb <<< "$s"
  d=/tmp/var/$PFX$vw$nv$mb; rm -rf $d; cp -r $SRC $d
  python - "$d/crvec_kernels.cuh" "$PAT" $vw $nv $mb <<'PY'
import re, sys
p, pat, vw, nv, mb = sys.argv[1:]
out = []
for l in open(p).read().split("\n"):
    if "struct KernelShape<" + pat + ">" in l:
        l = re.sub(r"vw = \d+, nv = \d+, minb = \d+", f"vw = {vw}, nv = {nv}, minb = {mb}", l)
    out.append(l)
open(p, "w").write("\n".join(out))
PY
  grep -c "KernelShape<$PAT> { static constexpr int vw = $vw, nv = $nv, minb = $mb" $d/crvec_kernels.cuh > /dev/null || echo "pattern $PAT not found"
done
for s in $4; do
  IFS=: read vw nv mb <<< "$s"
  python -m paper_2605_15547_b200.build --variant $PFX$vw$nv$mb /tmp/var/$PFX$vw$nv$mb > /tmp/var/$PFX$vw$nv$mb.log 2>&1 &
done
wait
for s in $4; do IFS=: read vw nv mb <<< "$s"; tail -n 1 /tmp/var/$PFX$vw$nv$mb.log; done
rm -rf paper_2605_15547_b200/variants/_build_*
