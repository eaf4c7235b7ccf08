"""TEST INFRASTRUCTURE ONLY -- build the C restatement (oracle/sv_ref.c) into oracle/libsvref.so.

Compiled for x86-64-v3 (AVX2/FMA) so the object built here also runs on the GPU box.
The reference itself is Python (rydsim); there is no C reference source to compile,
so no oracle/_ref is produced ("Oracle").
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sv_ref.c")
LIB = os.path.join(HERE, "libsvref.so")


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", "-o", LIB + ".tmp", SRC]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def load():
    import ctypes

    build()
    lib = ctypes.CDLL(LIB)
    dp = ctypes.POINTER(ctypes.c_double)
    lib.svref_matvec.argtypes = [ctypes.c_int, dp, dp, dp, dp]
    lib.svref_matvec.restype = None
    lib.svref_matvec_range.argtypes = [ctypes.c_int, dp, dp, dp, dp, ctypes.c_int64, ctypes.c_int64]
    lib.svref_matvec_range.restype = None
    lib.svref_build_diagonal.argtypes = [ctypes.c_int, dp, dp, dp]
    lib.svref_build_diagonal.restype = None
    lib.svref_fill.argtypes = [ctypes.c_int64, dp, ctypes.c_uint64]
    lib.svref_fill.restype = None
    lib.svref_threads.restype = ctypes.c_int
    lib.svref_set_threads.argtypes = [ctypes.c_int]
    lib.svref_set_threads.restype = None
    lib.svref_zdotc.argtypes = [ctypes.c_int64, dp, dp, dp]
    lib.svref_zdotc.restype = None
    lib.svref_zaxpy.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_double, dp, dp]
    lib.svref_zaxpy.restype = None
    lib.svref_zscal.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_double, dp, dp]
    lib.svref_zscal.restype = None
    lib.svref_norm2.argtypes = [ctypes.c_int64, dp]
    lib.svref_norm2.restype = ctypes.c_double
    return lib


if __name__ == "__main__":
    print(build(force=True))
