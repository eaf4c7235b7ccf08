"""Build the in-tree CUDA extension ``_rsv.so`` (sm_100a) with nvcc.

Used by ``__graft_entry__.build()`` and ``make``. The library is a plain C-ABI
shared object (include/rsv.h) loaded with ctypes; it links the CUDA runtime
statically so it does not depend on torch's bundled runtime version.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "rsv_kernels.cu"), os.path.join(HERE, "csrc", "rsv_capi.cu")]
HEADERS = [os.path.join(HERE, "csrc", "rsv_kernels.cuh"), os.path.join(ROOT, "include", "rsv.h")]
TARGET = os.path.join(HERE, "_rsv.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build() -> bool:
    if not os.path.exists(TARGET):
        return True
    t = os.path.getmtime(TARGET)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, target: str = TARGET, defines=()) -> str:
    if not force and target == TARGET and not needs_build():
        return TARGET
    cmd = [nvcc_path(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           *[f"-D{d}" for d in defines], "-o", target + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(TARGET)
