#!/bin/bash
# Developer: variants forcing one kernel shape (NV:MINB) and one rare-path form
# (RS = 0 register / 1 store) on every binary32 map kernel:
#   bash tools/mk_tune_variants.sh "2:3:0 2:3:1 ..."   -> variants t<NV><MINB><RS>
for s in $1; do
  IFS=: read nv mb rs <<< "$s"
  d=/tmp/var/t$nv$mb$rs; rm -rf $d; cp -r paper_2605_15547_b200/csrc $d
  python - "$d/crvec_kernels.cuh" $nv $mb $rs <<'PY'
import re, sys
p, nv, mb, rs = sys.argv[1:5]
s = open(p).read()
s = re.sub(r"static constexpr int vw = 4, nv = \d+, minb = \d+;", f"static constexpr int vw = 4, nv = {nv}, minb = {mb};", s)
s = s.replace("template <class F> struct RareStore { static constexpr bool value = false; };",
              "template <class F> struct RareStore { static constexpr bool value = %s; };" % ("true" if rs == "1" else "false"))
for t in ("template <int B> struct RareStore<FnLogB<B>>", "template <bool A> struct RareStore<FnAsinAcos<A>>",
          "template <> struct RareStore<FnCosh>", "template <> struct RareStore<FnTanh>"):
    s = re.sub(re.escape(t) + r" \{ static constexpr bool value = \w+; \};", "", s)
open(p, "w").write(s)
PY
done
for s in $1; do
  IFS=: read nv mb rs <<< "$s"
  python -m paper_2605_15547_b200.build --variant t$nv$mb$rs /tmp/var/t$nv$mb$rs > /tmp/var/t$nv$mb$rs.log 2>&1 &
done
wait
for s in $1; do IFS=: read nv mb rs <<< "$s"; tail -n 1 /tmp/var/t$nv$mb$rs.log; done
rm -rf paper_2605_15547_b200/variants/_build_*
