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


def _deps_newer(obj: str, src: str, csrc: str = CSRC) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    for f in os.listdir(csrc):
        if os.path.getmtime(os.path.join(csrc, f)) > t:
            return True
    return os.path.getmtime(os.path.join(ROOT, "include", "crvec.h")) > t


def build(force: bool = False, verbose: bool = False, csrc: str = CSRC, lib: str = LIB,
          build_dir: str = BUILD) -> str:
    """Compile the sources in `csrc` into `lib`. The defaults build the product
    library; other directories are developer A/B variants (loaded through the
    CRVEC_LIB environment variable by the perf tools)."""
    CSRC_, LIB_, BUILD_ = csrc, lib, build_dir
    os.makedirs(BUILD_, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC_, s))]
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for s in srcs:
            src = os.path.join(CSRC_, s)
            obj = os.path.join(BUILD_, s.replace(".cu", ".o"))
            objs.append(obj)
            if force or _deps_newer(obj, src, CSRC_):
                cmd = [nvcc(), *ARCH, *FLAGS, "-Xptxas", "-v", "-c", src, "-o", obj]
                jobs.append((s, ex.submit(subprocess.run, cmd, capture_output=True, text=True)))
        for s, fut in jobs:
            r = fut.result()
            with open(os.path.join(BUILD_, s + ".log"), "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {s}:\n{r.stderr[-4000:]}")
    if force or jobs or not os.path.exists(LIB_):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB_, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print("built", LIB_)
    return LIB_


def build_variant(name: str, csrc: str) -> str:
    """Developer A/B build: sources from `csrc` -> variants/libcrvec_<name>.so."""
    vdir = os.path.join(PKG, "variants")
    return build(verbose=True, csrc=csrc, lib=os.path.join(vdir, f"libcrvec_{name}.so"),
                 build_dir=os.path.join(vdir, "_build_" + name))


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        build_variant(sys.argv[i + 1], sys.argv[i + 2])
    else:
        build(force="--force" in sys.argv, verbose=True)
