"""Builds libhydro.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2403_14902_b200.build [--force] [--verbose]

The library links the NCCL that ships with torch (nvidia/nccl), so only one libnccl is
loaded next to torch's process group, and the CUDA runtime statically.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhydro.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("torch-bundled NCCL (nvidia/nccl) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "hydro.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def build(force: bool = False, verbose: bool = False, extra=(), out: str = None) -> str:
    """Compiles csrc/*.cu into libhydro.so (or `out` with extra nvcc flags, for A/B variants)."""
    lib_out = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    inc, lib = _nccl_dirs()
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *cus, "-o", lib_out + ".tmp",
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}", "-cudart", "static", *extra]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout + r.stderr, file=sys.stderr)
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", action="append", default=[],
                    help="NAME:FLAGS -> libhydro_NAME.so built with the extra nvcc flags (A/B experiments)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
    for v in a.variant:
        name, _, flags = v.partition(":")
        print(build(verbose=a.verbose, extra=tuple(flags.split()), out=os.path.join(HERE, f"libhydro_{name}.so")))
