"""Build libadop.so (the C-ABI library, include/adop.h) in-tree for sm_100a with nvcc.

    python -m paper_2110_06635_b200.build [--force]

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libadop.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-split-compile=0",  # the optimizer's work on the kernel instances in parallel threads
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "adop.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build LIB (or `out` with extra -D `defines`: tuning variants, e.g. ADOP_DSTAGES=3)."""
    if out is None and not force and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(PKG, "build" if out is None else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(bdir, exist_ok=True)
    logs = []
    procs = []
    for src in sources():  # the translation units compile concurrently
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for src, obj, p in procs:
        so, se = p.communicate()
        logs.append(so + se)
        if p.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    target = LIB if out is None else out
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs,
           "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, target)
    with open(os.path.join(bdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
