"""In-tree build of libqsocp_cuda.so (sm_100a only).

nvcc cross-compiles without a GPU; the resulting .so sits next to this file so
it travels with the repo snapshot to the GPU box.  No JIT, no fallback.
"""

from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libqsocp_cuda.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "--extended-lambda",
              "-fmad=false",  # keep the reference's mul-then-add rounding (no FMA contraction)
              "-Xcompiler", "-fPIC"]
CU = ["cone_kernels.cu", "kkt_kernels.cu", "spmv_kernels.cu", "ruiz_kernels.cu", "ldl.cu", "capi.cu"]
CPP = ["host_setup.cpp"]
FMA_OK = {"ldl.cu"}  # the factorisation is not a restatement of reference arithmetic: let it use FMA


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(HERE, "..", "include", "qsocp_cuda.h"))
    return hs


def build_library(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    jobs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(obj, [src] + hdrs):
            flags = [x for x in NVCC_FLAGS if not (f in FMA_OK and x == "-fmad=false")]
            if os.environ.get("QS_CONE_VARIANTS") and f == "cone_kernels.cu":  # tuning: slot-count instantiations
                flags = flags + ["-DQS_CONE_VARIANTS=" + os.environ["QS_CONE_VARIANTS"]]
            jobs.append([NVCC, *flags, "-c", src, "-o", obj])
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(obj, [src] + hdrs):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-pthread", "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")

    with ThreadPoolExecutor(max_workers=6) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, f + ".o") for f in CU + CPP]
    if force or jobs or _stale(LIB, objs):
        run([NVCC, "-shared", "-o", LIB, *objs, "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-pthread"])
    return LIB


if __name__ == "__main__":
    print(build_library(verbose=True))
