"""ctypes binding of the C ABI in ``include/rsv.h`` (the in-tree ``_rsv.so``).

The product path has no CPU fallback: importing works without a GPU (so the
CPU test-suite can check the exported symbols), but every compute call fails
loudly when the extension or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import RydsimError, SolverError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSV_LIB overrides the library path (used to A/B compile-time kernel variants in tools/)
LIB_PATH = os.environ.get("RSV_LIB") or os.path.join(_HERE, "_rsv.so")

RSV_OK = 0
RSV_ERR_ARG = -1
RSV_ERR_CUDA = -2
RSV_ERR_STATE = -3
RSV_ERR_NOT_CONVERGED = -4
RSV_DIAG_FLY = 1
RSV_DIAG_VEC = 2

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int_p = ctypes.POINTER(ctypes.c_int)
c_u64_p = ctypes.POINTER(ctypes.c_uint64)
c_ll_p = ctypes.POINTER(ctypes.c_longlong)


class KrylovReportC(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int),
        ("converged", ctypes.c_int),
        ("residual", ctypes.c_double),
        ("alpha0", ctypes.c_double),
        ("norm_in", ctypes.c_double),
        ("substeps", ctypes.c_int),
        ("matvecs", ctypes.c_int),
        ("regenerated", ctypes.c_int),
    ]


# rsv_comm_fn (include/rsv.h): int (*)(void* user, int op, int slot, int peer, double* host, int count)
COMM_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(ctypes.c_double), ctypes.c_int)
RSV_COMM_ALLREDUCE = 1
RSV_COMM_EXCHANGE_START = 2
RSV_COMM_EXCHANGE_WAIT = 3
RSV_COMM_ALLREDUCE_DEVICE = 4

# name -> (restype, argtypes); exactly the symbols declared in include/rsv.h
SIGNATURES = {
    "rsv_version": (ctypes.c_int, []),
    "rsv_last_error": (ctypes.c_char_p, []),
    "rsv_device_count": (ctypes.c_int, [c_int_p]),
    "rsv_create": (ctypes.c_int, [ctypes.c_int, c_double_p, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.POINTER(ctypes.c_void_p)]),
    "rsv_destroy": (None, [ctypes.c_void_p]),
    "rsv_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_bind_slots": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    "rsv_state_slot": (ctypes.c_int, [ctypes.c_void_p, c_int_p]),
    "rsv_bind_diag_vector": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "rsv_build_diagonal": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_void_p]),
    "rsv_state_modified": (ctypes.c_int, [ctypes.c_void_p]),
    "rsv_apply_hamiltonian": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "rsv_expm_step": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int, ctypes.c_double, c_double_p, c_double_p, ctypes.c_int,
                                     ctypes.POINTER(KrylovReportC)]),
    "rsv_set_observables": (ctypes.c_int, [ctypes.c_void_p, c_u64_p, ctypes.c_int]),
    "rsv_get_observables": (ctypes.c_int, [ctypes.c_void_p, c_double_p]),
    "rsv_measure": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p]),
    "rsv_observe": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, c_u64_p, ctypes.c_int, c_double_p,
                                   c_double_p]),
    "rsv_sample": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, c_double_p, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_int64), c_double_p]),
    "rsv_diff_norm_sq": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                        c_double_p]),
    "rsv_zdotc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, c_double_p]),
    "rsv_lanczos_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_uint64, c_double_p]),
    "rsv_axpy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                ctypes.c_double, ctypes.c_uint64]),
    "rsv_scale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_uint64]),
    "rsv_tridiag_exp_e1": (ctypes.c_int, [c_double_p, c_double_p, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                          c_double_p]),
    "rsv_pass_plan": (ctypes.c_int, [ctypes.c_void_p, c_int_p, ctypes.c_int]),
    "rsv_set_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]),
    "rsv_set_reorthogonalize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_tail_regeneration": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_shard_scratch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_speculation": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_fusion": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_shard": (ctypes.c_int, [ctypes.c_void_p, COMM_FN, ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_set_shard_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                          c_double_p, c_int_p]),
    "rsv_shard_local_norm_sq": (ctypes.c_int, [ctypes.c_void_p, c_double_p]),
    "rsv_enable_peer_access": (ctypes.c_int, [ctypes.c_void_p]),
    "rsv_shard_peer_stats": (ctypes.c_int, [ctypes.c_void_p, c_ll_p]),
    "rsv_set_shard_peers": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.c_int]),
    "rsv_set_profiling": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rsv_get_profile": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_ll_p]),
    "rsv_reset_profile": (ctypes.c_int, [ctypes.c_void_p]),
}

_lib = None
_lock = threading.Lock()


class NativeError(RydsimError):
    """The CUDA extension reported an error (or is missing)."""


def load():
    """Load ``_rsv.so`` once; raise NativeError if it is missing (no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"CUDA extension {LIB_PATH} is missing; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str = ""):
    if rc == RSV_OK:
        return
    msg = load().rsv_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == RSV_ERR_ARG:
        raise ValidationError(text)
    if rc == RSV_ERR_NOT_CONVERGED:
        raise SolverError(text)
    raise NativeError(text)


def dptr(arr):
    """ctypes double* for a contiguous float64 numpy array."""
    return arr.ctypes.data_as(c_double_p)


def tridiag_exp_e1(alphas, betas, tau, full=True):
    """exp(-1j tau T) e1 of the Lanczos tridiagonal through rsv_tridiag_exp_e1 (the step driver's own
    function; krylov.py:54). full=False returns only the last component (as a 1-element array)."""
    lib = load()
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    k = a.shape[0]
    b = np.ascontiguousarray(betas, dtype=np.float64)[: max(k - 1, 0)]
    out = np.zeros(2 * k if full else 2)
    rc = lib.rsv_tridiag_exp_e1(dptr(a), dptr(b) if k > 1 else None, k, float(tau), 1 if full else 0, dptr(out))
    check(rc, "rsv_tridiag_exp_e1")
    return out[0::2] + 1j * out[1::2]

