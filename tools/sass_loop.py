"""Static SASS census of a kernel's main loop (developer tool).

usage: python tools/sass_loop.py OBJ REGEX [--ne N]
Finds the functions whose mangled name matches REGEX in OBJ (cuobjdump -sass),
locates the longest backward branch (the grid-stride loop), and counts the
instructions inside it by mnemonic (per element when --ne is given). The loop
body includes the rare branch's code, so the hot count is reported both with
and without instructions the loop jumps over (straight-line fall-through).
"""
import collections
import re
import subprocess
import sys


def sass(obj, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def names(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    return re.findall(r"Function : (\S+)", out)


def census(ins):
    loops = []
    for a, t in ins:
        m = re.search(r"\bBRA\s+(?:`\(\.L_x_\d+\)|)?\s*(0x[0-9a-f]+)", t)
        if m and not t.startswith("@") or (m and "BRA" in t):
            tgt = int(m.group(1), 16) if m else None
            if tgt is not None and tgt < a:
                loops.append((a - tgt, tgt, a))
    if not loops:
        return None
    _, lo, hi = max(loops)
    body = [(a, t) for a, t in ins if lo <= a <= hi]
    # fall-through path: skip forward-branch targets' regions is hard; approximate
    # by excluding code after unconditional forward BRA until its target.
    hot = []
    skip_to = None
    for a, t in body:
        if skip_to is not None and a < skip_to:
            continue
        skip_to = None
        hot.append((a, t))
        m = re.match(r"(@!?U?P\w+\s+)?BRA(\.\w+)*\s+(?:`\(\.L_x_\d+\)\s*)?(0x[0-9a-f]+)", t)
        if m and m.group(1) is None:
            tgt = int(m.group(3), 16)
            if tgt > a:
                skip_to = tgt
    return body, hot


def op(t):
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    return t.split()[0]


def main():
    obj, rx = sys.argv[1], sys.argv[2]
    ne = int(sys.argv[sys.argv.index("--ne") + 1]) if "--ne" in sys.argv else 1
    for fn in names(obj):
        if not re.search(rx, fn):
            continue
        r = census(sass(obj, fn))
        if r is None:
            print(fn, "no loop")
            continue
        body, hot = r
        c = collections.Counter(op(t).split(".")[0] for _, t in hot)
        print(f"{fn}: loop {len(body)} instr, straight-line {len(hot)} -> {len(hot)/ne:.1f}/elem")
        print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(25)))


if __name__ == "__main__":
    main()
