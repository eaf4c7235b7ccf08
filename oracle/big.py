"""TEST INFRASTRUCTURE ONLY -- the reference's state-vector step at N = 27..30 on the host.

``sv_oracle.expm_multiply`` restates rydsim/krylov.py:67-125 with numpy, whose temporaries
(``w = w - c * v`` allocates a full vector) and single-threaded reductions make it unusable
at the headline sizes (8.6 GB per vector at N=29). This module runs the SAME loop --
same order of operations, full re-orthogonalisation, same convergence/breakdown tests,
same tridiagonal exponential (``sv_oracle.tridiag_exp_e1``) -- with the in-place OpenMP
vector operations of ``oracle/sv_ref.c`` and the C restatement of the compiled matvec
(rydsim/_kernels.py:13, dispatched by hamiltonian.py:180-187), so the GPU path can be
checked against the reference algorithm at N=27 (BASELINE configs[2]) and N=29
(configs[3]). Host memory: (k + 3) vectors of 16 * 2^N bytes plus the 8 * 2^N diagonal.

Pinning: ``svref_matvec`` is checked against the reference's golden H.psi vectors and this
loop against ``sv_oracle.expm_multiply`` (itself pinned to the reference's golden Lanczos
steps) in tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import build as _build
from .sv_oracle import BREAKDOWN_RTOL, NS_TO_US, OracleError, tridiag_exp_e1

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _build.load()
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class HostHamiltonian:
    """The slice of one step (sv.py:116,127-129): diagonal built once, matvec by the C kernel."""

    def __init__(self, omegas, deltas, u):
        self.omegas = np.ascontiguousarray(omegas, dtype=np.float64)
        self.n = len(self.omegas)
        self.half = np.ascontiguousarray(0.5 * self.omegas)
        self.diag = np.empty(1 << self.n)
        lib().svref_build_diagonal(self.n, _p(np.ascontiguousarray(deltas, dtype=np.float64)),
                                   _p(np.ascontiguousarray(u, dtype=np.float64)), _p(self.diag))

    def matvec(self, psi, out):
        """out = H psi (hamiltonian.py:164 apply_hamiltonian -> _kernels.py:13)."""
        lib().svref_matvec(self.n, _p(psi), _p(self.diag), _p(self.half), _p(out))
        return out

    def matvec_range(self, psi, out, b0, b1):
        lib().svref_matvec_range(self.n, _p(psi), _p(self.diag), _p(self.half), _p(out), int(b0), int(b1))
        return out


def vdot(x, y):
    r = np.zeros(2)
    lib().svref_zdotc(x.size, _p(x), _p(y), _p(r))
    return complex(r[0], r[1])


def axpy(a, x, y):
    """y += a x."""
    a = complex(a)
    lib().svref_zaxpy(x.size, a.real, a.imag, _p(x), _p(y))


def scal(a, x, y):
    a = complex(a)
    lib().svref_zscal(x.size, a.real, a.imag, _p(x), _p(y))


def norm(x):
    return math.sqrt(lib().svref_norm2(x.size, _p(x)))


def expm_multiply(ham: HostHamiltonian, psi, dt_ns, tolerance=1e-10, max_krylov_dim=100,
                  norm_epsilon=1e-14, max_vectors=None, consume_input=False):
    """exp(-i dt 1e-3 H) psi by the reference's Lanczos loop (krylov.py:67-125), line by line:

    norm / early returns (krylov.py:86-91), basis[0] = psi/||psi|| (:94), w = H v_j (:100),
    alpha = Re <v_j|w> (:101), w -= alpha v_j, w -= beta_{j-1} v_{j-1} (:102-103), full
    re-orthogonalisation against every basis vector in order (:104-105), beta = ||w|| (:106),
    y = exp(-i tau T) e1 (:108), residual and breakdown tests (:109-114), the Krylov cap
    (:115-116), out = norm_in * sum y_i v_i (:119-122).

    Returns (out, iterations, converged, residual, alphas, betas). ``max_vectors`` bounds the
    host memory (raises OracleError instead of exhausting it); ``consume_input`` normalises
    ``psi`` in place as basis[0] (one vector less of host memory; ``psi`` is overwritten).
    """
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    norm_in = norm(psi)
    if norm_in <= norm_epsilon:
        return psi.copy(), 0, True, 0.0, [], []
    if dt_ns == 0.0:
        return psi.copy(), 1, True, 0.0, [], []
    tau = dt_ns * NS_TO_US
    v0 = psi if consume_input else np.empty_like(psi)
    scal(1.0 / norm_in, psi, v0)
    basis = [v0]
    alphas, betas = [], []
    converged = False
    residual = math.inf
    while True:
        w = np.empty_like(psi)
        ham.matvec(basis[-1], w)
        a = vdot(basis[-1], w).real
        alphas.append(a)
        axpy(-a, basis[-1], w)
        if betas:
            axpy(-betas[-1], basis[-2], w)
        for v in basis:
            axpy(-vdot(v, w), v, w)
        b = norm(w)
        y = tridiag_exp_e1(alphas, betas, tau)
        residual = b * abs(y[-1])
        scale = max(1.0, max(abs(x) for x in alphas), max(betas, default=0.0))
        if residual <= tolerance or b <= BREAKDOWN_RTOL * scale:
            converged = True
            del w
            break
        if len(alphas) >= max_krylov_dim:
            del w
            break
        if max_vectors is not None and len(basis) >= max_vectors:
            raise OracleError(f"host Lanczos needs more than {max_vectors} basis vectors")
        betas.append(b)
        scal(1.0 / b, w, w)
        basis.append(w)
    out = np.zeros_like(basis[0])
    for coef, v in zip(y, basis):
        axpy(coef, v, out)
    scal(norm_in, out, out)
    return out, len(alphas), converged, float(residual), alphas, betas
