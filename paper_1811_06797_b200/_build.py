"""Build libigalr.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import re
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


# Spill guard: the canonical kernels on the bulk-copy + resident-y path (the ones
# every BASELINE config runs: k_canon<..., YRES=true, TMA=true, ...>) sit near the 255-register
# cliff, where ptxas flips between 0 and 300+ bytes of spills on unrelated edits.  A build whose
# ptxas reports spills in one of them fails instead of shipping a silently slower kernel.
# (Other variants - odd extents, per-round y staging - may spill a few bytes; they are reported.)
SPILL_RE = re.compile(r"Registers are spilled to local memory in function '([^']+)', (\d+) bytes spill stores, "
                      r"(\d+) bytes spill loads")
GUARDED = re.compile(r"k_canon.*ELb1ELb1ELb[01]ELb[01]EEEv")
# Ratchet: guarded variants (k_canon<Shape, P, LW, 2, QX, YRES=1, TMA=1, SPLIT, PACK>) that spill in
# the current build, with their byte counts (stores, loads).  Any other guarded spill, or growth of
# these, fails the build.  The BASELINE kernels: c3 stiffness/mass (P 3, LW 16, QX 4) spill nothing;
# c4 stiffness (P 3, LW 12, QX 2, split, packed) nothing, c4 mass (packed) 8 B (one double, since
# the x-coefficients of single-round plans stay in registers for a whole segment: measured -1.4 % on c4); c5 stiffness and mass (P 4, LW 13, QX 4) nothing.
_MK = "_ZN5igalr2f27k_canonINS0_%sELi%dELi%dELi2ELi%dELb1ELb1ELb%dELb%dEEEvNS0_5Args2ENS0_6KSplitE"
KNOWN_SPILLS = {
    _MK % ("10ShapeMassKILi4EE", 3, 12, 2, 0, 1): (8, 8),  # c4 mass (packed): one double, per-segment x-coefficients
    _MK % ("10ShapeMassKILi4EE", 3, 16, 1, 0, 0): (20, 28),
    _MK % ("10ShapeMassKILi4EE", 3, 16, 2, 0, 0): (16, 20),
    _MK % ("10ShapeMassKILi4EE", 3, 16, 2, 0, 1): (20, 28),
    _MK % ("10ShapeMassKILi4EE", 3, 16, 4, 0, 1): (20, 28),
    _MK % ("11ShapeStiffA", 3, 12, 2, 1, 0): (52, 72),
    _MK % ("11ShapeStiffA", 3, 16, 1, 0, 1): (4, 4),
    _MK % ("11ShapeStiffA", 3, 16, 1, 1, 1): (52, 72),
    _MK % ("11ShapeStiffA", 3, 16, 2, 0, 1): (4, 4),
    _MK % ("11ShapeStiffA", 3, 16, 2, 1, 0): (60, 80),
    _MK % ("11ShapeStiffA", 3, 16, 2, 1, 1): (44, 60),
    _MK % ("11ShapeStiffA", 3, 16, 4, 0, 1): (4, 4),
    _MK % ("11ShapeStiffA", 3, 16, 4, 1, 1): (44, 60),
    _MK % ("10ShapeMassKILi3EE", 4, 12, 2, 0, 0): (64, 80),
    _MK % ("10ShapeMassKILi3EE", 4, 12, 4, 0, 0): (68, 88),
    _MK % ("10ShapeMassKILi4EE", 4, 12, 1, 0, 0): (32, 32),
    _MK % ("10ShapeMassKILi4EE", 4, 12, 2, 0, 0): (108, 108),
    _MK % ("10ShapeMassKILi4EE", 4, 12, 4, 0, 0): (100, 100),
    _MK % ("10ShapeMassKILi4EE", 4, 13, 4, 0, 0): (92, 92),
}


def check_spills(log: str):
    bad = []
    for m in SPILL_RE.finditer(log):
        name, st, ld = m.group(1), int(m.group(2)), int(m.group(3))
        ks, kl = KNOWN_SPILLS.get(name, (0, 0))
        if GUARDED.search(name) and (st > ks or ld > kl):
            bad.append("%s (%d B stores, %d B loads)" % (name, st, ld))
    if bad:
        raise RuntimeError("ptxas spilled registers in guarded production kernels:\n  " + "\n  ".join(bad))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise subprocess.CalledProcessError(r.returncode, cmd[0])
    return r.stdout + r.stderr


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
        logs = list(ex.map(_run, jobs))
    try:
        check_spills("".join(logs))
    except RuntimeError:
        for j in jobs:  # force a rebuild next time (the objects exist but must not ship)
            try:
                os.remove(j[-1])
            except OSError:
                pass
        raise
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
