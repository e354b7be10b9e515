"""Build libfse_b200.so in-tree (sm_100a) with nvcc.

    python -m paper_2204_14193_b200.build      # or __graft_entry__.build()

The shared library is the product: CUDA kernels (csrc/*.cu) + the C ABI
(csrc/api.cpp, include/fse_b200.h).  No torch types cross the ABI; the
library is loaded with ctypes by paper_2204_14193_b200/_lib.py.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SO = os.path.join(HERE, "libfse_b200.so")
SOURCES = ["csrc/generic.cu", "csrc/fast.cu", "csrc/fast_small.cu", "csrc/fast_mid.cu", "csrc/spatial.cu",
           "csrc/api.cpp"]
DEPS = SOURCES + ["csrc/common.cuh", "csrc/dft.cuh", "csrc/kernels.h", "../include/fse_b200.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(os.path.join(HERE, d)) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """Compile the library.  `defines`/`out` build diagnostic variants
    (e.g. FSE_DIAG) next to the product library; the product is SO."""
    target = os.path.abspath(out) if out else SO
    if not force and out is None and up_to_date():
        return SO
    cmd = [nvcc(), *ARCH, *[f"-D{d}" for d in defines], "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "-I", os.path.join(REPO, "include"),
           "-o", target + ".tmp", *[os.path.join(HERE, s) for s in SOURCES]]
    if out is not None:  # diagnostic variants may try other code-generation flags
        cmd[1:1] = os.environ.get("FSE_NVCC_EXTRA", "").split()
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
