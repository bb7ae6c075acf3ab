"""Per-mnemonic executed-instruction census of an ncu capture (developer tool).

usage: python tools/ncu_sass.py REP.ncu-rep ELEMENTS [--top N]
Reads `ncu -i REP --page source --csv --print-source sass` and reports, per
SASS mnemonic, warp instructions executed per element x 32 (thread-instructions
per element) and the stall samples attributed to it, plus the hottest lines.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))


def main():
    rep, n = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    rs = rows(rep)
    by = collections.Counter()
    st = collections.Counter()
    stall_cols = [c for c in rs[0] if c.startswith("stall_") and "Not Issued" not in c]
    stalls = collections.Counter()
    tot = 0
    for r in rs:
        src = r["Source"].strip()
        m = re.sub(r"^@!?U?P\w+\s+", "", src).split()
        if not m:
            continue
        mn = m[0].split(".")[0]
        ex = float(r["Instructions Executed"] or 0)
        by[mn] += ex
        tot += ex
        st[mn] += float(r["Warp Stall Sampling (All Samples)"] or 0)
        for c in stall_cols:
            stalls[c] += float(r[c] or 0)
    print(f"total {tot*32/n:.2f} thread-instr/elem ({tot:.0f} warp instr)")
    for k, v in by.most_common(top):
        print(f"  {k:10s} {v*32/n:7.2f}/elem   stall samples {st[k]:.0f}")
    s = sum(stalls.values())
    print("stall mix:", ", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in stalls.most_common(10)))
    if "--lines" in sys.argv:
        hot = sorted(rs, key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
        for r in hot:
            print(f"  {r['Warp Stall Sampling (All Samples)']:>6} {float(r['Instructions Executed'] or 0)*32/n:6.3f}  {r['Source'].strip()}")


if __name__ == "__main__":
    main()
