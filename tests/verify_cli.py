"""crvec verification CLI (the SPEC's verify module, ref: SPEC.md:233-307; the
reference's proj/src/verify.cpp and tools/crvec.cpp are stubs).

  python tests/verify_cli.py verify   --fn expf --mode all [--stride 1] [--range LO:HI] [--report R.json]
  python tests/verify_cli.py corpus   --fn log  --file PATH [--all-modes]
  python tests/verify_cli.py callouts --fn log  --uniform 0.5:2.0 --n 10000000 [--seed S]

verify --stride 1 without a range runs the exhaustive 2^32 GPU sweep against
the golden chunk hashes and re-checks any mismatching chunk element by element
against the oracle; strided / ranged runs evaluate the selected patterns on the
GPU and compare every element with the oracle. Reports are deterministic JSON
(VerifyReport: fn, modes, inputs tested, mismatches with ulp distance,
coverage, wall time). Lives under tests/ because it executes the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_15547_b200 as crvec  # noqa: E402
from oracle import oracle as O  # noqa: E402

MODES = {"rne": 0, "rz": 1, "ru": 2, "rd": 3}


def ulp32_distance(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """ref: proj/src/fpbits.cpp:189-209 (ordered32 difference); NaN -> -1."""
    def ordered(u):
        u = u.astype(np.int64)
        mag = u & 0x7FFFFFFF
        return np.where(u >> 31, -mag - 1, mag)
    d = np.abs(ordered(a) - ordered(b))
    nan = ((a << 1) > 0xFF000000) | ((b << 1) > 0xFF000000)
    return np.where(nan, -1, d)


def gpu_eval(name: str, xbits: np.ndarray, mode: int) -> np.ndarray:
    import torch
    t = torch.from_numpy(xbits.view(np.float32)).cuda()
    out = crvec.eval_f32(name, t, mode)
    if isinstance(out, tuple):
        return tuple(o.cpu().numpy().view(np.uint32) for o in out)
    return out.cpu().numpy().view(np.uint32)


def compare(name, x, modes, report, cap=100):
    outs = [("sin", "cos")] if name == "sincosf" else [crvec.ORACLE_NAME[name]]
    for m in modes:
        got = gpu_eval(name, x, m)
        got = got if isinstance(got, tuple) else (got,)
        for g, ofn in zip(got, outs[0] if name == "sincosf" else outs):
            want = O.f32(ofn, x, m)
            bad = np.nonzero(g != want)[0]
            report["mismatch_count"] += int(len(bad))
            for i in bad[: max(0, cap - len(report["mismatches"]))]:
                report["mismatches"].append({
                    "input": f"0x{int(x[i]):08x}", "mode": m, "fn": ofn, "got": f"0x{int(g[i]):08x}",
                    "expected": f"0x{int(want[i]):08x}",
                    "ulp": int(ulp32_distance(np.array([g[i]]), np.array([want[i]]))[0])})
    report["inputs_tested"] += int(len(x))


def cmd_verify(a):
    t0 = time.time()
    modes = list(range(4)) if a.mode == "all" else [MODES[a.mode]]
    rep = {"fn": a.fn, "modes": modes, "inputs_tested": 0, "mismatch_count": 0, "mismatches": []}
    if a.stride == 1 and not a.range:
        rep["coverage"] = "exhaustive 2^32 (GPU sweep vs golden chunk hashes; mismatching chunks re-checked)"
        h, h2, _ = crvec.sweep_f32(a.fn)
        golds = [("sin", h), ("cos", h2)] if a.fn == "sincosf" else [(crvec.ORACLE_NAME[a.fn], h)]
        for g, arr in golds:
            gold = np.load(os.path.join(ROOT, "tests", "golden", "sweep", g + ".npy"))
            bad_chunks = np.nonzero((gold[:, modes] != arr[:, modes]).any(axis=1))[0]
            rep.setdefault("mismatching_chunks", []).extend(int(c) for c in bad_chunks)
            for c in bad_chunks[:4]:
                x = np.arange(int(c) << 20, (int(c) + 1) << 20, dtype=np.uint64).astype(np.uint32)
                compare(a.fn, x, modes, rep)
        rep["inputs_tested"] = 2 ** 32
    else:
        lo, hi = (int(v, 0) for v in a.range.split(":")) if a.range else (0, 2 ** 32 - 1)
        x = np.arange(lo, hi + 1, a.stride, dtype=np.uint64).astype(np.uint32)
        rep["coverage"] = f"patterns [{lo:#x}, {hi:#x}] stride {a.stride}"
        for i in range(0, len(x), 1 << 22):
            compare(a.fn, x[i:i + (1 << 22)], modes, rep)
    rep["wall_s"] = round(time.time() - t0, 3)
    out = json.dumps(rep, indent=1)
    if a.report:
        open(a.report, "w").write(out)
    print(out)
    return 1 if rep["mismatch_count"] or rep.get("mismatching_chunks") else 0


def parse_corpus(path):
    """`<hex-float>[,<hex-float-expected>]` per line, '#' comments (ref: SPEC.md:289)."""
    recs, diags = [], []
    for ln, line in enumerate(open(path), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        try:
            parts = [p.strip() for p in line.split(",")]
            recs.append((ln, float.fromhex(parts[0]), float.fromhex(parts[1]) if len(parts) > 1 else None))
        except ValueError as e:
            diags.append({"line": ln, "error": str(e)})
    return recs, diags


def cmd_corpus(a):
    recs, diags = parse_corpus(a.file)
    modes = list(range(4)) if a.all_modes else [0]
    x = np.array([r[1] for r in recs], np.float64)
    rep = {"fn": a.fn, "file": a.file, "records": len(recs), "parse_errors": diags,
           "kernel_mismatches": [], "corpus_oracle_disagreements": []}
    rng = np.random.default_rng(0)
    for m in modes:
        if a.fn in ("exp2", "log"):
            # randomized co-resident lanes around each record (SPEC corpus_check)
            pad = rng.uniform(0.5, 2, len(x) * 31)
            xx = np.concatenate([x, pad])
            got = crvec._f64(a.fn, xx, m, None)[: len(x)].view(np.uint64)
            want = O.f64(a.fn, x.view(np.uint64), m)
        else:
            xb = x.astype(np.float32).view(np.uint32)
            got = gpu_eval(a.fn, xb, m)
            want = O.f32(crvec.ORACLE_NAME[a.fn], xb, m)
        for i in np.nonzero(got != want)[0]:
            rep["kernel_mismatches"].append({"line": recs[i][0], "mode": m, "got": hex(int(got[i])),
                                             "expected": hex(int(want[i]))})
        if m == 0:
            for i, r in enumerate(recs):
                if r[2] is not None:
                    exp_bits = np.array([r[2]]).view(np.uint64)[0] if a.fn in ("exp2", "log") else \
                        np.array([r[2]], np.float32).view(np.uint32)[0]
                    if exp_bits != want[i]:
                        rep["corpus_oracle_disagreements"].append({"line": r[0]})
    print(json.dumps(rep, indent=1))
    return 1 if rep["kernel_mismatches"] else 0


def cmd_callouts(a):
    lo, hi = (float(v) for v in a.uniform.split(":"))
    rng = np.random.default_rng(a.seed)
    x = rng.uniform(lo, hi, a.n)
    st = crvec.FastPathStats()
    crvec._f64(a.fn, x, 0, st)
    rep = {"fn": a.fn, "distribution": f"uniform({lo}, {hi})", "n": a.n, "seed": a.seed,
           "undecided": st.undecided, "rate": st.undecided / a.n,
           "rate_log2": float(np.log2(st.undecided / a.n)) if st.undecided else None,
           "accurate_undecided": st.accurate_undecided, "host_callouts": st.host_callouts}
    print(json.dumps(rep, indent=1))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="crvec")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("--fn", required=True, choices=list(crvec.FN_IDS))
    v.add_argument("--mode", default="rne", choices=list(MODES) + ["all"])
    v.add_argument("--stride", type=int, default=1)
    v.add_argument("--range")
    v.add_argument("--report")
    c = sub.add_parser("corpus")
    c.add_argument("--fn", required=True)
    c.add_argument("--file", required=True)
    c.add_argument("--all-modes", action="store_true")
    k = sub.add_parser("callouts")
    k.add_argument("--fn", required=True, choices=["exp2", "log"])
    k.add_argument("--uniform", required=True)
    k.add_argument("--n", type=int, default=10_000_000)
    k.add_argument("--seed", type=int, default=1)
    a = ap.parse_args(argv)
    return {"verify": cmd_verify, "corpus": cmd_corpus, "callouts": cmd_callouts}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
