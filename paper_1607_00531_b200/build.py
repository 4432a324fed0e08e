"""Build libepicorr_b200.so in-tree with nvcc for sm_100a.

Arithmetic flags are part of the contract: -fmad=false plus the default
IEEE-rounded division/sqrt make every restated reference expression round
exactly like the reference's -O3 -ffp-contract=off build.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libepicorr_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["api.cu", "bstep.cu", "zstep.cu", "aux_kernels.cu", "gn.cu", "pcg.cu", "slab.cu", "multilevel.cu", "image.cu",
           "admm_f32.cu", "operators_t2.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
         "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-rdc=false", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


# the fp32 variant has no bitwise contract: contraction to FMA is allowed there
FMAD_ON = {"admm_f32.cu"}
LIBS = ["-lcudart"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".inc"))]
    return hs + [os.path.join(ROOT, "include", "epicorr_b200.h")]


def _compile(src, verbose):
    out = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + _headers()
    if not _stale(out, deps):
        return out
    flags = [f for f in FLAGS if not (src in FMAD_ON and f == "-fmad=false")]
    if src in FMAD_ON:
        flags.append("-fmad=true")
    cmd = [NVCC, *ARCH, *flags, "-Xptxas", "-v" if verbose else "-O3", "-c",
           os.path.join(CSRC, src), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return out


def build(verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if force:
        for s in srcs:
            o = os.path.join(OBJ, os.path.splitext(s)[0] + ".o")
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, *LIBS]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
