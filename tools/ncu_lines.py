"""Developer: thread-instructions executed per element by CUDA source line
(ncu --page source --print-source cuda,sass of a -lineinfo build).
usage: python tools/ncu_lines.py REP.ncu-rep ELEMENTS [--top N]"""
import csv
import io
import subprocess
import sys


def main():
    rep, n = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fpath = [], "?"
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1].split("/")[-1]
            continue
        if r[0] and r[0].isdigit() and len(r) > 9:
            try:
                rows.append((float(r[8]) / n, fpath, int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot = sum(x[0] for x in rows)
    print(f"total {tot:.2f} thread-instr/elem over {len(rows)} source lines")
    for v, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{v:7.2f}  {f}:{ln:<5d} {src[:110]}")


if __name__ == "__main__":
    main()
