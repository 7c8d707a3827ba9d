"""Build libigalr.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.environ.get("IGALR_LIB_OUT", os.path.join(HERE, "libigalr.so"))
BUILD = os.environ.get("IGALR_BUILD_DIR", os.path.join(ROOT, "build", "igalr"))
EXTRA = os.environ.get("IGALR_NVCC_EXTRA", "").split()  # experiment defines (never set for the product)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]

SOURCES = ["abi.cu", "factors.cu", "apply_unfused.cu", "apply_fused.cu", "apply_fused2.cu", "canon_p3.cu",
           "canon_p4.cu", "kkt.cu", "minres.cu", "prec.cu", "weights.cu", "tt.cu"]


def _newer(src_paths, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_paths)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "iga_lr.h"))
    objs = []
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer([src] + headers + [__file__], obj):
            cmd = [NVCC] + ARCH + FLAGS + EXTRA + ["-I" + INCLUDE, "-I" + CSRC, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            jobs.append(cmd)
    # translation units compile in parallel (the canonical-kernel units dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for rc in ex.map(subprocess.call, jobs):
            if rc != 0:
                raise subprocess.CalledProcessError(rc, "nvcc")
    if force or _newer(objs, LIB):
        tmp = LIB + ".tmp.%d" % os.getpid()
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-cudart=static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
