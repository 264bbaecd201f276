"""Build libss.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libss.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # FMAs only where the contract writes them (inline PTX)
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-shared",
]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]


def _deps():
    files = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    files.append(os.path.join(INCLUDE, "ss.h"))
    return files


def lib_path(variant: str | None = None) -> str:
    return LIB if not variant else os.path.join(PKG, "libss_%s.so" % variant)


def up_to_date(path: str = LIB) -> bool:
    if not os.path.exists(path):
        return False
    t = os.path.getmtime(path)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines=()) -> str:
    """Compile libss.so; ``variant`` + ``defines`` build a tuning variant
    libss_<variant>.so of the same sources (tools/kbench.py)."""
    out = lib_path(variant)
    if up_to_date(out) and not force:
        return out
    tmp = out + ".tmp%d" % os.getpid()
    cmd = ["nvcc", *NVCC_FLAGS, *["-D" + d for d in defines], "-I", INCLUDE, "-I", CSRC,
           "-o", tmp, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libss.so")
    with open(os.path.join(PKG, "build_ptxas%s.log" % ("_" + variant if variant else "")), "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
