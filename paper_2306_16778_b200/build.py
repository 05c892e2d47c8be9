"""Build libpfx.so (the C-ABI library, include/pfx.h) in-tree with nvcc for sm_100a.

Usage: python -m paper_2306_16778_b200.build   (or build() from __graft_entry__)
Objects go to paper_2306_16778_b200/build/, the library to paper_2306_16778_b200/libpfx.so.
Rebuilds only when a source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUTDIR = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libpfx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
# timing experiments only (e.g. PFX_NVCC_FLAGS=-DPFX_TRI_EXP=1 ablates a kernel phase)
COMMON += os.environ.get("PFX_NVCC_FLAGS", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


STAMP = LIB + ".flags"


def _flags_id() -> str:
    """Everything that changes the generated code besides the sources: the nvcc command
    line (including PFX_NVCC_FLAGS ablations) and the compiler."""
    return " ".join([NVCC, *ARCH, *COMMON])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    # a library built with different flags (e.g. an interrupted timing ablation that
    # compiled a phase out) is never reused
    try:
        with open(STAMP) as fh:
            if fh.read() != _flags_id():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def _compile(src: str) -> str:
    obj = os.path.join(OUTDIR, os.path.basename(src) + ".o")
    if src.endswith(".cpp"):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *COMMON, "-Xptxas", "-v", "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    with open(obj + ".log", "w") as fh:
        fh.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OUTDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        objs = list(pool.map(_compile, _sources()))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "--cudart=static", "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as fh:
        fh.write(_flags_id())
    if verbose:
        for o in objs:
            print(open(o + ".log").read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
