"""Build libcrvec.so (sm_100a) in-tree with nvcc.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false:
--fmad=false is the CUDA analogue of the reference's -ffp-contract=off
(ref: proj/CMakeLists.txt:16-18): every fused multiply-add in the kernels is an
explicit __fma_rn, nothing is contracted behind our back. No fast-math, no FTZ.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libcrvec.so")
BUILD = os.path.join(PKG, "_build")
SOURCES = ["crvec_api.cu", "crvec_fam_exp.cu", "crvec_fam_log.cu", "crvec_fam_trig.cu",
           "crvec_fam_atrig.cu", "crvec_f64.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=default", "-I", os.path.join(ROOT, "include")]
if os.path.exists(os.path.join(CSRC, "crvec_f64.cu")):
    FLAGS.append("-DCRVEC_WITH_F64")


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps_newer(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return os.path.getmtime(os.path.join(ROOT, "include", "crvec.h")) > t


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for s in srcs:
            src = os.path.join(CSRC, s)
            obj = os.path.join(BUILD, s.replace(".cu", ".o"))
            objs.append(obj)
            if force or _deps_newer(obj, src):
                cmd = [nvcc(), *ARCH, *FLAGS, "-Xptxas", "-v", "-c", src, "-o", obj]
                jobs.append((s, ex.submit(subprocess.run, cmd, capture_output=True, text=True)))
        for s, fut in jobs:
            r = fut.result()
            with open(os.path.join(BUILD, s + ".log"), "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {s}:\n{r.stderr[-4000:]}")
    if force or jobs or not os.path.exists(LIB):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
