"""Measurements on device-resident states -- mirror of rydsim/observables.py (dense-state part).

``occupations`` (observables.py:82), ``occupation`` (:95), ``correlation`` (:102),
``overlap`` (:120), ``norm_difference`` (:137), ``fidelity`` (:157), ``sample_bitstrings`` (:167),
``ObservableSpec`` (:221) and ``ObservableRecord`` (:263) with the reference's
names and validation. The reductions run in the rsv kernels: an observable is a
bit mask M with value sum_b |psi_b|^2 [b & M == M] / sum_b |psi_b|^2.
The MPS representation is out of scope.

Extension (north star): kind ``"energy"`` records <psi|H_k|psi> / <psi|psi> for
the slice H_k that produced the state (conserved by the step, so it is the
first Lanczos coefficient of that step times 1 -- no extra pass).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ValidationError

__all__ = [
    "ObservableSpec",
    "ObservableRecord",
    "occupation",
    "occupations",
    "correlation",
    "overlap",
    "norm_difference",
    "fidelity",
    "qubit_count",
    "format_bitstring",
    "occupation_masks",
    "sample_bitstrings",
]

_SAMPLE_BATCH = 4096       # observables.py:34
_NORM_TOLERANCE = 1e-6     # observables.py:35


def sample_uniforms(shots: int, seed: int) -> np.ndarray:
    """The reference's uniform draws (observables.py:194-213): one PCG64 child stream of
    SeedSequence(seed) per batch of 4096 shots, so the samples do not depend on the execution."""
    batches = [min(_SAMPLE_BATCH, shots - start) for start in range(0, shots, _SAMPLE_BATCH)]
    streams = np.random.SeedSequence(seed).spawn(len(batches))
    out = np.empty(shots, dtype=np.float64)
    pos = 0
    for count, stream in zip(batches, streams):
        out[pos:pos + count] = np.random.Generator(np.random.PCG64(stream)).random(count)
        pos += count
    return out


def sample_bitstrings(state, shots: int, seed: int, renormalize: bool = False) -> np.ndarray:
    """Basis-state indices drawn from |amplitude|^2 (observables.py:167, dense path), on the device:
    the state never leaves HBM (inverse CDF: chunk sums -> prefix -> one warp per shot)."""
    if shots < 1:
        raise ValidationError(f"shots must be >= 1, got {shots}")
    n = qubit_count(state)
    x = _dev(state)
    u = sample_uniforms(int(shots), int(seed))
    out = np.empty(int(shots), dtype=np.int64)
    nsq = ctypes.c_double()
    ctx = _ctx(n)
    nat.check(ctx.lib.rsv_sample(ctx.ctx, x.data_ptr(), nat.dptr(u), int(shots),
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(nsq)),
              "rsv_sample")
    norm = math.sqrt(max(0.0, nsq.value))
    if abs(norm - 1.0) > _NORM_TOLERANCE and not renormalize:
        raise ValidationError(f"state norm deviates from 1 by {abs(norm - 1.0):.3e}; "
                              "pass renormalize=True to sample anyway")
    return out


def qubit_count(state) -> int:
    size = int(state.shape[0]) if hasattr(state, "shape") else len(state)
    n = int(round(math.log2(size))) if size > 0 else -1
    if n < 0 or 2 ** n != size:
        raise ValidationError(f"dense state length {size} is not a power of 2")
    return n


def _dev(state):
    from .hamiltonian import _as_device

    return _as_device(state)[0]


def _ctx(n):
    from .hamiltonian import context_for

    ctx = context_for(n, np.zeros((n, n)))
    ctx.sync_stream()
    return ctx


def occupation_masks(n, qubits=()):
    qs = list(qubits) if qubits else list(range(n))
    return [1 << q for q in qs]


def _observe(state, masks):
    n = qubit_count(state)
    x = _dev(state)
    ctx = _ctx(n)
    arr = np.ascontiguousarray(np.asarray(masks, dtype=np.uint64))
    out = np.zeros(max(1, arr.size))
    nsq = ctypes.c_double()
    nat.check(ctx.lib.rsv_observe(ctx.ctx, x.data_ptr(), arr.ctypes.data_as(nat.c_u64_p), int(arr.size),
                                  nat.dptr(out), ctypes.byref(nsq)), "rsv_observe")
    return out[: arr.size]


def occupations(state) -> np.ndarray:
    """<n_q> for every qubit (probabilities renormalised, observables.py:82-92)."""
    n = qubit_count(state)
    return _observe(state, occupation_masks(n))


def occupation(state, qubit: int) -> float:
    n = qubit_count(state)
    if not 0 <= qubit < n:
        raise ValidationError(f"qubit {qubit} out of range for N={n}")
    return float(_observe(state, [1 << qubit])[0])


def correlation(state, qi: int, qj: int) -> float:
    """<n_qi n_qj> for two distinct qubits (observables.py:102)."""
    n = qubit_count(state)
    if not (0 <= qi < n and 0 <= qj < n):
        raise ValidationError(f"qubits ({qi}, {qj}) out of range for N={n}")
    if qi == qj:
        raise ValidationError("correlation needs two distinct qubits; use occupation")
    return float(_observe(state, [(1 << qi) | (1 << qj)])[0])


def overlap(state_a, state_b) -> complex:
    """<a|b> (observables.py:120)."""
    na, nb = qubit_count(state_a), qubit_count(state_b)
    if na != nb:
        raise ValidationError(f"qubit counts differ: {na} vs {nb}")
    a, b = _dev(state_a), _dev(state_b)
    ctx = _ctx(na)
    out = (ctypes.c_double * 2)()
    nat.check(ctx.lib.rsv_zdotc(ctx.ctx, a.data_ptr(), b.data_ptr(), a.numel(), out))
    return complex(out[0], out[1])


def norm_difference(state_a, state_b) -> float:
    """||a - b||_2, global phase included (observables.py:137), without cancellation."""
    na, nb = qubit_count(state_a), qubit_count(state_b)
    if na != nb:
        raise ValidationError(f"qubit counts differ: {na} vs {nb}")
    a, b = _dev(state_a), _dev(state_b)
    ctx = _ctx(na)
    out = ctypes.c_double()
    nat.check(ctx.lib.rsv_diff_norm_sq(ctx.ctx, a.data_ptr(), b.data_ptr(), a.numel(), ctypes.byref(out)))
    return math.sqrt(max(0.0, out.value))


def fidelity(state_a, state_b) -> float:
    """|<a|b>|^2 (observables.py:157)."""
    return float(abs(overlap(state_a, state_b)) ** 2)


def format_bitstring(index: int, n_qubits: int) -> str:
    """Character k (from the left) is qubit k (observables.py:162)."""
    return "".join(str((index >> q) & 1) for q in range(n_qubits))


@dataclass(frozen=True)
class ObservableSpec:
    """What to measure and how often (observables.py:221).

    kind: "occupation" (qubits: labels, empty = all), "correlation" (flat pair
    list) or "energy" (extension). every_n_steps = 0 means final step only.
    """

    kind: str
    qubits: tuple = ()
    every_n_steps: int = 1

    def __post_init__(self):
        if self.kind not in ("occupation", "correlation", "energy"):
            raise ValidationError(f"unknown observable kind {self.kind!r}")
        object.__setattr__(self, "qubits", tuple(int(q) for q in self.qubits))
        if self.every_n_steps < 0:
            raise ValidationError("every_n_steps must be >= 0")
        if self.kind == "correlation" and (len(self.qubits) == 0 or len(self.qubits) % 2):
            raise ValidationError("correlation needs a flat, even-length list of qubit pairs")

    def due(self, step: int, total_steps: int) -> bool:
        if self.every_n_steps == 0:
            return step == total_steps
        return step % self.every_n_steps == 0

    def masks(self, n: int):
        if self.kind == "occupation":
            return occupation_masks(n, self.qubits)
        if self.kind == "correlation":
            out = []
            for i, j in zip(self.qubits[::2], self.qubits[1::2]):
                if not (0 <= i < n and 0 <= j < n) or i == j:
                    raise ValidationError(f"bad correlation pair ({i}, {j}) for N={n}")
                out.append((1 << i) | (1 << j))
            return out
        return []


@dataclass
class ObservableRecord:
    spec_index: int
    kind: str
    qubits: tuple
    step: int
    t_ns: float
    values: list = field(default_factory=list)
