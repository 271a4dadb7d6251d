"""Build libnmfb.so (sm_100a) in-tree with nvcc.

    python -m paper_1506_08938_b200.build [--verbose]

Compiles every csrc/*.cu for ``-gencode arch=compute_100a,code=sm_100a`` with
``-lineinfo`` (ncu source view) and links a plain C-ABI shared library
(static cudart, no torch linkage).  Incremental: a .cu is recompiled only when
it or a header is newer than its object.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# NMFB_BUILD_DIR / NMFB_EXTRA_FLAGS: an experiment variant of the library
# built elsewhere (load it with NMFB_LIB_PATH); the default build is in-tree
_VAR = os.environ.get("NMFB_BUILD_DIR")
OBJ = os.path.join(_VAR, "obj") if _VAR else os.path.join(PKG, "_build")
LIB = os.path.join(_VAR, "libnmfb.so") if _VAR else os.path.join(PKG, "libnmfb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", os.path.join(REPO, "include"),
         *os.environ.get("NMFB_EXTRA_FLAGS", "").split()]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(REPO, "include", "*.h"))


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or hdr_mtime > t


def build(verbose=False, ptxas_info=False):
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr = max((os.path.getmtime(h) for h in _headers()), default=0.0)
    jobs = []
    for src in srcs:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if _stale(src, obj, hdr):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        return res.stderr

    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
            for err in pool.map(run, jobs):
                if verbose and err:
                    print(err)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if jobs or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
