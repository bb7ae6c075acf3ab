"""Summarise tools/gpu_inst.sh output: per kernel, thread-instructions per
element, registers, achieved occupancy and issue activity (ncu, one launch
each; n = 2^28 binary32 / 2^26 binary64 elements as in tools/perf.py)."""
import csv
import re
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
by = {}
for r in rows:
    k = (r["ID"], r["Kernel Name"])
    by.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"].replace(",", "")
print(f"{'kernel':34s} {'instr/elem':>10s} {'regs':>5s} {'occ%':>6s} {'issue%':>7s} {'us':>8s}")
for (i, name), m in by.items():
    fn = re.sub(r"^void crvec::|\(.*$", "", name)
    n = 2**26 if "k_f64" in name else 2**28
    inst = float(m.get("smsp__inst_executed.sum", 0)) * 32 / n
    print(f"{fn[:34]:34s} {inst:10.2f} {m.get('launch__registers_per_thread', '?'):>5s} "
          f"{float(m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0)):6.1f} "
          f"{float(m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0)):7.1f} "
          f"{float(m.get('gpu__time_duration.sum', 0))/1e3:8.1f}")
