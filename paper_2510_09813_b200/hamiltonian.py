"""Rydberg Hamiltonian in structured form -- mirror of rydsim/hamiltonian.py on B200.

Same names, argument meaning and errors as the reference:
``Register`` (hamiltonian.py:43), ``interaction_matrix`` (:66), ``weighted_bit_sum``
(:83), ``interaction_diagonal`` (:99), ``build_diagonal`` (:114), ``HamiltonianSlice``
(:125), ``apply_hamiltonian`` (:164), ``build_dense`` (:191). Bit order: qubit i = bit i
of the basis index.

Differences by design (B200-first):
* a slice built with ``HamiltonianSlice.from_parameters`` keeps (omegas, deltas, U):
  the lo pass of the CUDA matvec computes the diagonal on the fly (``diag='vec'``
  reads a precomputed float64 interaction diagonal instead); ``slice.diagonal`` is
  still the reference's 2^N array, built on the GPU the first time it is read;
* the 2^N diagonals (``weighted_bit_sum``, ``interaction_diagonal``,
  ``build_diagonal``) are built by a device kernel and returned as numpy arrays like
  the reference's (``device=True`` keeps the CUDA tensor);
* states may be complex128 CUDA tensors (results stay on the device) or numpy
  arrays (copied in, result copied back: the "e2e" path).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as nat
from .errors import ValidationError

__all__ = [
    "Register",
    "interaction_matrix",
    "weighted_bit_sum",
    "interaction_diagonal",
    "build_diagonal",
    "HamiltonianSlice",
    "apply_hamiltonian",
    "build_dense",
    "DENSE_QUBIT_CAP",
]

DENSE_QUBIT_CAP = 14


@dataclass(frozen=True)
class Register:
    """Atom positions (um, 2D or 3D) and the interaction constant C (hamiltonian.py:43)."""

    positions_um: tuple
    interaction_c: float

    def __post_init__(self):
        pts = tuple(tuple(float(x) for x in p) for p in self.positions_um)
        object.__setattr__(self, "positions_um", pts)
        if len(pts) < 1:
            raise ValidationError("register needs at least one atom")
        dims = {len(p) for p in pts}
        if not dims <= {2, 3} or len(dims) != 1:
            raise ValidationError(f"positions must all be 2D or all 3D, got dimensions {sorted(dims)}")

    @property
    def qubit_count(self) -> int:
        return len(self.positions_um)


def interaction_matrix(reg: Register) -> np.ndarray:
    """U_ij = C / |r_i - r_j|^6, zero diagonal; coincident atoms rejected (hamiltonian.py:66).

    N x N host work (N <= 48); the 2^N work happens on the GPU.
    """
    pos = np.asarray(reg.positions_um, dtype=float)
    diff = pos[:, None, :] - pos[None, :, :]
    d2 = (diff ** 2).sum(-1)
    n = len(pos)
    iu = np.triu_indices(n, 1)
    if n > 1 and np.any(d2[iu] == 0.0):
        k = int(np.argmax(d2[iu] == 0.0))
        raise ValidationError(f"atoms {iu[0][k]} and {iu[1][k]} coincide")
    u = np.zeros((n, n))
    u[iu] = reg.interaction_c / d2[iu] ** 3
    return u + u.T


def _torch():
    import torch

    return torch


@lru_cache(maxsize=8)
def _context(n: int, u_bytes: bytes, diag: str, device_index: int):
    from .engine import Context

    u = np.frombuffer(u_bytes, dtype=np.float64).reshape(n, n)
    return Context(n, u, diag=diag, device=f"cuda:{device_index}")


def context_for(n: int, u: np.ndarray, diag: str = "fly"):
    torch = _torch()
    if not torch.cuda.is_available():
        raise nat.NativeError("no CUDA device: the state-vector hot path has no CPU fallback")
    u = np.ascontiguousarray(u, dtype=np.float64)
    return _context(int(n), u.tobytes(), diag, torch.cuda.current_device())


def _device_diagonal(deltas, u, device):
    """-sum delta_i n_i + sum_{i<j} U_ij n_i n_j by the device kernel (rsv_build_diagonal)."""
    deltas = np.ascontiguousarray(deltas, dtype=np.float64)
    torch = _torch()
    ctx = context_for(len(deltas), u)
    out = torch.empty(1 << len(deltas), dtype=torch.float64, device=ctx.device)
    ctx.sync_stream()
    nat.check(ctx.lib.rsv_build_diagonal(ctx.ctx, nat.dptr(deltas), out.data_ptr()), "rsv_build_diagonal")
    return out if device else out.cpu().numpy()


def weighted_bit_sum(weights, device: bool = False):
    """v[b] = sum_i weights[i] bit_i(b), length 2^N (hamiltonian.py:83)."""
    w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
    return _device_diagonal(-w, np.zeros((len(w), len(w))), device)


def interaction_diagonal(u: np.ndarray, device: bool = False):
    """d[b] = sum_{i<j} U_ij bit_i(b) bit_j(b) (hamiltonian.py:99)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.ndim != 2 or u.shape[0] != u.shape[1]:
        raise ValidationError(f"interaction matrix must be square, got shape {u.shape}")
    return _device_diagonal(np.zeros(u.shape[0]), u, device)


def build_diagonal(deltas, u: np.ndarray, device: bool = False):
    """Full diagonal -sum delta_i n_i + sum_{i<j} U_ij n_i n_j (hamiltonian.py:114); numpy like the
    reference, or the CUDA tensor with ``device=True``."""
    deltas = np.ascontiguousarray(deltas, dtype=np.float64)
    if u.shape != (len(deltas), len(deltas)):
        raise ValidationError(
            f"interaction matrix shape {u.shape} does not match {len(deltas)} detunings")
    return _device_diagonal(deltas, u, device)


class HamiltonianSlice:
    """One piecewise-constant Hamiltonian (hamiltonian.py:125).

    ``HamiltonianSlice(omegas, diagonal)`` is the reference's explicit-diagonal form
    (diagonal: 2^N float64, numpy or CUDA tensor). ``from_parameters(omegas, deltas, u)``
    keeps the structured form used by the hot path (diagonal on the fly); its ``.diagonal``
    is materialised (on the GPU, returned as numpy) the first time it is read.
    """

    def __init__(self, omegas, diagonal=None, deltas=None, interaction=None):
        omegas = np.ascontiguousarray(omegas, dtype=float)
        n = len(omegas)
        self.omegas = omegas
        self.deltas = None
        self.interaction = None
        self._diagonal = None
        if diagonal is None:
            if deltas is None or interaction is None:
                raise ValidationError("slice needs a diagonal or (deltas, interaction)")
            self.deltas = np.ascontiguousarray(deltas, dtype=float)
            self.interaction = np.ascontiguousarray(interaction, dtype=float)
            if self.interaction.shape != (n, n) or self.deltas.shape != (n,):
                raise ValidationError(
                    f"interaction matrix shape {self.interaction.shape} does not match {n} detunings")
        else:
            if isinstance(diagonal, (list, tuple)):
                diagonal = np.asarray(diagonal, dtype=float)
            elif isinstance(diagonal, np.ndarray):
                diagonal = np.ascontiguousarray(diagonal, dtype=float)
            size = int(diagonal.shape[0]) if len(diagonal.shape) else -1
            if size != 2 ** n or len(diagonal.shape) != 1:
                raise ValidationError(f"diagonal has length {tuple(diagonal.shape)}, expected 2^{n}")
            self._diagonal = diagonal

    @property
    def qubit_count(self) -> int:
        return len(self.omegas)

    @property
    def structured(self) -> bool:
        """True when the slice carries (deltas, U): the matvec computes the diagonal on the fly."""
        return self.deltas is not None

    @property
    def diagonal(self):
        """The 2^N diagonal (hamiltonian.py:131); built on the GPU on first access for structured slices."""
        if self._diagonal is None:
            self._diagonal = build_diagonal(self.deltas, self.interaction)
        return self._diagonal

    @classmethod
    def from_parameters(cls, omegas, deltas, u: np.ndarray) -> "HamiltonianSlice":
        omegas = np.asarray(omegas, dtype=float)
        deltas = np.asarray(deltas, dtype=float)
        u = np.asarray(u, dtype=float)
        if u.shape != (len(deltas), len(deltas)):
            raise ValidationError(
                f"interaction matrix shape {u.shape} does not match {len(deltas)} detunings")
        return cls(omegas, None, deltas, u)

    def dense_diagonal(self):
        """The 2^N diagonal as a CUDA tensor."""
        if self._diagonal is not None:
            return _as_device(self._diagonal, dtype="float64")[0]
        return build_diagonal(self.deltas, self.interaction, device=True)

    def __repr__(self):
        form = "structured" if self.structured else "explicit diagonal"
        return f"HamiltonianSlice(N={self.qubit_count}, {form})"


def _as_device(x, dtype="complex128"):
    """(cuda tensor, was_numpy)."""
    torch = _torch()
    tdt = getattr(torch, dtype)
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.dtype(dtype))).to("cuda"), True
    if not x.is_cuda:
        return x.to(device="cuda", dtype=tdt), True
    return x.to(tdt).contiguous(), False


def apply_hamiltonian(slice_: HamiltonianSlice, psi, out=None, force_numpy: bool = False):
    """H @ psi without materialising H (hamiltonian.py:164) -- the CUDA bit-group passes.

    psi: complex CUDA tensor (or numpy array: copied in, result copied back). ``force_numpy``
    is accepted for call compatibility and changes nothing: the reference uses it to select
    its sequential numpy loop for cross-checks; this package has one (CUDA) implementation
    and no CPU path (both reference paths agree with it to 1e-12, tests/test_gpu_parity.py).
    """
    n = slice_.qubit_count
    torch = _torch()
    x, was_numpy = _as_device(psi)
    if tuple(x.shape) != (2 ** n,):
        raise ValidationError(f"state has shape {tuple(x.shape)}, expected ({2 ** n},)")
    if slice_.structured:
        ctx = context_for(n, slice_.interaction, "fly")
        deltas = slice_.deltas
        diag_tensor = None
    else:
        ctx = context_for(n, np.zeros((n, n)), "vec")
        deltas = np.zeros(n)
        diag_tensor = _as_device(slice_._diagonal, dtype="float64")[0]
    y = out if (out is not None and not was_numpy) else torch.empty_like(x)
    if y.data_ptr() == x.data_ptr() and n > 12:
        y = torch.empty_like(x)
    ctx.sync_stream()
    if diag_tensor is not None:
        nat.check(ctx.lib.rsv_bind_diag_vector(ctx.ctx, diag_tensor.data_ptr(), 0))
    nat.check(ctx.lib.rsv_apply_hamiltonian(ctx.ctx, nat.dptr(slice_.omegas), nat.dptr(deltas),
                                            x.data_ptr(), y.data_ptr()), "rsv_apply_hamiltonian")
    if out is not None and not was_numpy and y.data_ptr() != out.data_ptr():
        out.copy_(y)
        y = out
    if was_numpy:
        res = y.cpu().numpy()
        if out is not None:
            out[...] = res
            return out
        return res
    return y


def build_dense(slice_: HamiltonianSlice) -> np.ndarray:
    """Dense 2^N x 2^N matrix, small-N checking helper only (hamiltonian.py:191)."""
    n = slice_.qubit_count
    if n > DENSE_QUBIT_CAP:
        raise ValidationError(
            f"dense Hamiltonian refused for N={n} > {DENSE_QUBIT_CAP} "
            "(exponential memory); use the structured apply instead")
    dim = 2 ** n
    # the diagonal from the GPU (build_diagonal, or the slice's explicit one); the off-diagonal
    # entries are the constants Omega_i/2 at (b, b ^ 2^i), placed as the reference places them
    # (round 1 built H column by column from 2^N GPU matvecs)
    diag = slice_.diagonal
    diag = diag.cpu().numpy() if hasattr(diag, "cpu") else np.asarray(diag)
    h = np.zeros((dim, dim), dtype=complex)
    rows = np.arange(dim)
    h[rows, rows] = diag
    for i in range(n):
        h[rows, rows ^ (1 << i)] += 0.5 * float(slice_.omegas[i])
    return h
