"""crvec verification CLI (the SPEC's verify module, ref: SPEC.md:233-307; the
reference's proj/src/verify.cpp and tools/crvec.cpp are stubs).

  python tests/verify_cli.py verify   --fn expf --mode all [--stride 1] [--range LO:HI] [--report R.json]
  python tests/verify_cli.py corpus   --fn log  --file PATH [--all-modes]
  python tests/verify_cli.py callouts --fn log  --uniform 0.5:2.0 --n 10000000 [--seed S]
  python tests/verify_cli.py consistency --fn expf --n 1000000 [--seed S]
  python tests/verify_cli.py exactness

--jobs N sets the host threads of the oracle comparisons (default: all cores);
the GPU side needs none. Every command prints one JSON document (the
VerifyReport schema above) and a one-line human summary on stderr.

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


JOBS = 0  # oracle threads (0 = all host cores)


def compare(name, x, modes, report, cap=100):
    outs = [("sin", "cos")] if name == "sincosf" else [crvec.ORACLE_NAME[name]]
    for m in modes:
        got = gpu_eval(name, x, m)
        got = got if isinstance(got, tuple) else (got,)
        for g, ofn in zip(got, outs[0] if name == "sincosf" else outs):
            want = O.f32(ofn, x, m, threads=JOBS)
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


def cmd_consistency(a):
    """consistency_check (ref: SPEC.md verify module): for n seeded random lanes
    (half uniform bit patterns, half the function's interesting range), the
    device-pointer path equals the host-pointer path, array results equal the
    scalar entry point lane by lane, results do not depend on the array's
    alignment / length split (element offsets 1..3 take the scalar head and a
    different vector phase), and a subset equals the oracle (the reference
    backend here)."""
    import torch
    rng = np.random.default_rng(a.seed)
    from tests.inputs import RANGES
    lo, hi = RANGES[a.fn]
    x = np.concatenate([rng.integers(0, 2 ** 32, a.n // 2, dtype=np.uint64).astype(np.uint32),
                        rng.uniform(lo, hi, a.n - a.n // 2).astype(np.float32).view(np.uint32)])
    rep = {"fn": a.fn, "n": int(a.n), "seed": a.seed, "checks": {}}
    ok = True
    for m in range(4):
        xf = x.view(np.float32)
        host = crvec.eval_f32(a.fn, xf, m)
        dev = crvec.eval_f32(a.fn, torch.from_numpy(xf).cuda(), m)
        host = host if isinstance(host, tuple) else (host,)
        dev = dev if isinstance(dev, tuple) else (dev,)
        same = all(np.array_equal(h.view(np.uint32), d.cpu().numpy().view(np.uint32)) for h, d in zip(host, dev))
        rep["checks"][f"device_vs_host_mode{m}"] = same
        ok &= same
        # alignment / split independence: the same lanes at element offsets 1..3
        for off in (1, 2, 3):
            buf = torch.empty(a.n + off, dtype=torch.float32, device="cuda")
            buf[off:] = torch.from_numpy(xf).cuda()
            o = crvec.eval_f32(a.fn, buf[off:], m)
            o = o if isinstance(o, tuple) else (o,)
            same = all(np.array_equal(h.view(np.uint32), d.cpu().numpy().view(np.uint32)) for h, d in zip(host, o))
            rep["checks"][f"offset{off}_mode{m}"] = same
            ok &= same
        # array vs scalar entry point (single-output functions)
        if a.fn != "sincosf":
            sc = getattr(crvec, "cr_" + a.fn + "_scalar")
            idx = rng.integers(0, a.n, 64)
            same = all(np.float32(sc(float(xf[i]), m)).view(np.uint32) == host[0].view(np.uint32)[i]
                       or (np.isnan(xf[i]) and np.isnan(host[0][i])) for i in idx)
            rep["checks"][f"array_vs_scalar_mode{m}"] = bool(same)
            ok &= bool(same)
        # subset vs the oracle
        sub = x[:: max(1, a.n // 65536)]
        outs = ("sin", "cos") if a.fn == "sincosf" else (crvec.ORACLE_NAME[a.fn],)
        got = crvec.eval_f32(a.fn, sub.view(np.float32), m)
        got = got if isinstance(got, tuple) else (got,)
        same = all(np.array_equal(g.view(np.uint32), O.f32(f, sub, m, threads=JOBS)) for g, f in zip(got, outs))
        rep["checks"][f"oracle_subset_mode{m}"] = same
        ok &= same
    rep["pass"] = bool(ok)
    print(json.dumps(rep, indent=1))
    return 0 if ok else 1


def cmd_exactness(a):
    """Exactness suite (ref: SPEC.md acceptance #5): algebraically exact
    results in every mode — exp2f / exp2 on integers (normal and subnormal
    powers of two), log2f on powers of two, log(1) = +0 — plus the other exact
    cases the binary32 functions have (exp/expm1/sinh/tanh/sin/tan/asin/atan
    of +-0, cos(0) = cosh(0) = 1, log/log10/log1p of 1 / 10^k / 0, rsqrt of
    4^k), each compared with the oracle as well as with the exact value."""
    rep = {"checks": {}, "fn": "all"}
    ok = True
    ints = np.arange(-149, 128, dtype=np.float32)
    p2 = np.array([2.0 ** k for k in range(-149, 128)], dtype=np.float32)
    p10 = np.array([10.0 ** k for k in range(0, 11)], dtype=np.float32)
    p4 = np.array([4.0 ** k for k in range(-74, 64)], dtype=np.float32)
    zeros = np.array([0.0, -0.0], dtype=np.float32)
    for m in range(4):
        c = {
            "exp2f(int)": np.array_equal(crvec.cr_exp2f(ints, m), np.ldexp(np.float32(1), ints.astype(int))),
            "log2f(2^k)": np.array_equal(crvec.cr_log2f(p2, m), np.arange(-149, 128, dtype=np.float32)),
            "exp2(int)": np.array_equal(crvec.cr_exp2(np.arange(-1074, 1024, dtype=np.float64), m),
                                        np.ldexp(1.0, np.arange(-1074, 1024))),
            "log(1)=+0": bool(crvec.cr_log(np.array([1.0]), m)[0] == 0.0 and
                              not np.signbit(crvec.cr_log(np.array([1.0]), m)[0])),
            "log10f(10^k)": np.array_equal(crvec.cr_log10f(p10, m), np.arange(0, 11, dtype=np.float32)),
            "rsqrtf(4^k)": np.array_equal(crvec.cr_rsqrtf(p4, m), (1.0 / np.sqrt(p4.astype(np.float64))).astype(np.float32)),
            "cos/cosh(0)=1": bool((crvec.cr_cosf(zeros, m) == 1).all() and (crvec.cr_coshf(zeros, m) == 1).all()),
        }
        for name in ("expm1f", "sinhf", "tanhf", "sinf", "tanf", "asinf", "atanf", "log1pf"):
            r = getattr(crvec, "cr_" + name)(zeros, m)
            c[f"{name}(+-0)"] = bool(np.array_equal(r.view(np.uint32), zeros.view(np.uint32)))
        for k, v in c.items():
            rep["checks"][f"{k}_mode{m}"] = bool(v)
            ok &= bool(v)
        for name in crvec.F32_FUNCS:  # the same exact inputs through the oracle
            xs = np.concatenate([ints, p2, p10, p4, zeros]).view(np.uint32)
            got = crvec.eval_f32(name, xs.view(np.float32), m).view(np.uint32)
            same = np.array_equal(got, O.f32(crvec.ORACLE_NAME[name], xs, m, threads=JOBS))
            rep["checks"][f"{name}_oracle_mode{m}"] = same
            ok &= same
    rep["pass"] = bool(ok)
    print(json.dumps(rep, indent=1))
    return 0 if ok else 1


def main(argv=None):
    ap = argparse.ArgumentParser(prog="crvec")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("--fn", required=True, choices=list(crvec.FN_IDS))
    v.add_argument("--mode", default="rne", choices=list(MODES) + ["all"])
    v.add_argument("--stride", type=int, default=1)
    v.add_argument("--range")
    v.add_argument("--report")
    v.add_argument("--jobs", type=int, default=0, help="oracle host threads (0 = all cores)")
    c = sub.add_parser("corpus")
    c.add_argument("--fn", required=True)
    c.add_argument("--file", required=True)
    c.add_argument("--all-modes", action="store_true")
    k = sub.add_parser("callouts")
    k.add_argument("--fn", required=True, choices=["exp2", "log"])
    k.add_argument("--uniform", required=True)
    k.add_argument("--n", type=int, default=10_000_000)
    k.add_argument("--seed", type=int, default=1)
    q = sub.add_parser("consistency")
    q.add_argument("--fn", required=True, choices=list(crvec.FN_IDS))
    q.add_argument("--n", type=int, default=1_000_000)
    q.add_argument("--seed", type=int, default=1)
    sub.add_parser("exactness")
    a = ap.parse_args(argv)
    if not hasattr(a, "fn"):
        a.fn = "all"
    global JOBS
    JOBS = getattr(a, "jobs", 0) or 0
    rc = {"verify": cmd_verify, "corpus": cmd_corpus, "callouts": cmd_callouts,
          "consistency": cmd_consistency, "exactness": cmd_exactness}[a.cmd](a)
    print(f"crvec {a.cmd} --fn {a.fn}: {'PASS' if rc == 0 else 'FAIL'}", file=sys.stderr)
    return rc


if __name__ == "__main__":
    sys.exit(main())
