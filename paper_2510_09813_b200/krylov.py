"""Lanczos exp(-i dt H) psi -- mirror of rydsim/krylov.py on B200.

``KrylovConfig`` (krylov.py:28), ``KrylovReport`` (krylov.py:47) and
``expm_multiply(matvec, psi, dt_ns, cfg)`` (krylov.py:67) keep the reference's
names, defaults, validation and convergence rule
(|beta_k [exp(-i tau T_k)]_{k,1}| <= tolerance, breakdown beta <= 1e-14 scale).

Two device paths:
* ``matvec`` is a ``HamiltonianSlice`` -> the fused B200 step (rsv_expm_step):
  the Lanczos recurrence, alpha/beta reductions and normalisation live inside
  the H.psi passes; no re-orthogonalisation pass ("Lanczos
  fusion" for why the results agree with the reference to the tolerance);
* ``matvec`` is any callable on CUDA tensors -> a device Lanczos built from the
  rsv vector kernels with the reference's full re-orthogonalisation.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _native as nat
from .errors import ValidationError

__all__ = ["KrylovConfig", "KrylovReport", "expm_multiply", "NS_TO_US"]

NS_TO_US = 1e-3
_BREAKDOWN_RTOL = 1e-14


@dataclass(frozen=True)
class KrylovConfig:
    tolerance: float = 1e-10
    max_krylov_dim: int = 100
    norm_epsilon: float = 1e-14
    # extension: re-orthogonalise every Lanczos vector against the basis as the reference does
    # (krylov.py:103-104); the fused default is the plain three-term recurrence
    reorthogonalize: bool = False

    def __post_init__(self):
        if not 0.0 < self.tolerance <= 1e-1:
            raise ValidationError(f"krylov tolerance must be in (0, 0.1], got {self.tolerance}")
        if self.max_krylov_dim < 2:
            raise ValidationError(f"max_krylov_dim must be >= 2, got {self.max_krylov_dim}")


@dataclass
class KrylovReport:
    iterations: int
    converged: bool
    residual: float
    substeps: int = 1
    alpha0: float = float("nan")
    norm_in: float = float("nan")
    matvecs: int = 0
    regenerated: int = 0   # Lanczos vectors recomputed because the basis outgrew the resident slots


def _tridiag_exp_e1(alphas, betas, tau):
    """exp(-1j tau T) e1 on the host (krylov.py:54), by the step driver's own routine (rsv_tridiag_exp_e1)."""
    return nat.tridiag_exp_e1(alphas, betas, tau)


def _fused(slice_, psi, dt_ns, cfg):
    from .engine import SvEngine
    from .hamiltonian import _as_device

    n = slice_.qubit_count
    x, was_numpy = _as_device(psi)
    if tuple(x.shape) != (2 ** n,):
        raise ValidationError(f"state has shape {tuple(x.shape)}, expected ({2 ** n},)")
    from .engine import free_device_bytes

    # leave room for the returned vector next to the workspace (at large N it takes all of HBM)
    budget = max(0, free_device_bytes(x.device) - (16 << n) - (1 << 30))
    if slice_.structured:
        eng = SvEngine(n, slice_.interaction, diag="fly", max_krylov_dim=cfg.max_krylov_dim,
                       device=x.device, memory_budget_bytes=budget)
        deltas = slice_.deltas
    else:
        eng = SvEngine(n, np.zeros((n, n)), diag="vec", max_krylov_dim=cfg.max_krylov_dim, device=x.device,
                       memory_budget_bytes=budget)
        eng.dvec.copy_(_as_device(slice_.diagonal, dtype="float64")[0])
        deltas = np.zeros(n)
    try:
        eng.set_reorthogonalize(getattr(cfg, "reorthogonalize", False))   # absent on the reference's config
        eng.set_state(x)
        rep = eng.step(slice_.omegas, deltas, float(dt_ns), cfg.tolerance, cfg.max_krylov_dim, cfg.norm_epsilon)
        out = eng.state().clone()
    finally:
        eng.close()
    report = KrylovReport(rep.iterations, bool(rep.converged), float(rep.residual), 1 + rep.substeps,
                          rep.alpha0, rep.norm_in, rep.matvecs, rep.regenerated)
    return (out.cpu().numpy() if was_numpy else out), report


def _generic(matvec, psi, dt_ns, cfg):
    """Reference algorithm (krylov.py:82-125) with device vectors and rsv vector kernels."""
    import torch

    from .hamiltonian import _as_device, context_for

    x, was_numpy = _as_device(psi)
    x = x.reshape(-1)
    nelem = x.numel()
    ctx = context_for(1, np.zeros((1, 1)))
    ctx.sync_stream()
    lib = ctx.lib

    def zdot(a, b):
        out = (ctypes.c_double * 2)()
        nat.check(lib.rsv_zdotc(ctx.ctx, a.data_ptr(), b.data_ptr(), nelem, out))
        return complex(out[0], out[1])

    norm_in = math.sqrt(max(0.0, zdot(x, x).real))
    if norm_in <= cfg.norm_epsilon:
        out = x.clone()
        return (out.cpu().numpy() if was_numpy else out), KrylovReport(0, True, 0.0)
    if dt_ns == 0.0:
        out = x.clone()
        return (out.cpu().numpy() if was_numpy else out), KrylovReport(1, True, 0.0)
    tau = dt_ns * NS_TO_US
    v0 = torch.empty_like(x)
    nat.check(lib.rsv_scale(ctx.ctx, v0.data_ptr(), x.data_ptr(), 1.0 / norm_in, 0.0, nelem))
    basis = [v0]
    alphas, betas = [], []
    converged = False
    residual = math.inf
    y = np.array([1.0 + 0.0j])
    while True:
        w = matvec(basis[-1])
        w = _as_device(w)[0].reshape(-1).clone()
        alpha = zdot(basis[-1], w).real
        alphas.append(alpha)
        nsq = ctypes.c_double()
        prev = basis[-2] if betas else None
        nat.check(lib.rsv_lanczos_update(ctx.ctx, w.data_ptr(), basis[-1].data_ptr(),
                                         prev.data_ptr() if prev is not None else None, alpha,
                                         betas[-1] if betas else 0.0, nelem, ctypes.byref(nsq)))
        for v in basis:   # full re-orthogonalisation (krylov.py:103-104)
            c = zdot(v, w)
            nat.check(lib.rsv_axpy(ctx.ctx, w.data_ptr(), v.data_ptr(), -c.real, -c.imag, nelem))
        beta = math.sqrt(max(0.0, zdot(w, w).real))
        y = _tridiag_exp_e1(alphas, betas, tau)
        residual = beta * abs(y[-1])
        k = len(alphas)
        scale = max(1.0, max(abs(a) for a in alphas), max(betas, default=0.0))
        if residual <= cfg.tolerance or beta <= _BREAKDOWN_RTOL * scale:
            converged = True
            break
        if k >= cfg.max_krylov_dim:
            break
        betas.append(beta)
        nxt = torch.empty_like(w)
        nat.check(lib.rsv_scale(ctx.ctx, nxt.data_ptr(), w.data_ptr(), 1.0 / beta, 0.0, nelem))
        basis.append(nxt)
    out = torch.zeros_like(x)
    for coeff, v in zip(y, basis):
        c = complex(coeff) * norm_in
        nat.check(lib.rsv_axpy(ctx.ctx, out.data_ptr(), v.data_ptr(), c.real, c.imag, nelem))
    torch.cuda.current_stream().synchronize()
    rep = KrylovReport(iterations=len(alphas), converged=converged, residual=float(residual))
    return (out.cpu().numpy() if was_numpy else out), rep


def expm_multiply(matvec, psi, dt_ns: float, cfg: KrylovConfig = KrylovConfig()):
    """Return (exp(-1j * dt * 1e-3 * H) @ psi, report) via Lanczos (krylov.py:67)."""
    from .hamiltonian import HamiltonianSlice

    if isinstance(matvec, HamiltonianSlice):
        return _fused(matvec, psi, dt_ns, cfg)
    if not callable(matvec):
        raise ValidationError("matvec must be a HamiltonianSlice or a callable")
    return _generic(matvec, psi, dt_ns, cfg)
