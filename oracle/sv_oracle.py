"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the rydsim state-vector path.

Every function names the reference function (``/root/reference/pkg/src/rydsim/<file>:<line>``)
whose behaviour it restates. Conventions shared with the reference
(hamiltonian.py:1-8): qubit i is bit i of the basis index (qubit 0 = LSB);
energies in rad/us, times in ns, positions in um; dt*H phases use the single
factor 1e-3 (krylov.py:21).

The GPU product never imports this module (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.interpolate import CubicSpline

NS_TO_US = 1e-3                 # krylov.py:21
BREAKDOWN_RTOL = 1e-14          # krylov.py:25
ASSUMED_KRYLOV_DIM_SV = 15      # sv.py:40
DEFAULT_INTERACTION_C = 5_000_000.0   # generator.py:23
DEFAULT_SPACING_UM = 7.0              # generator.py:24
TWO_PI = 2.0 * math.pi


class OracleError(Exception):
    pass


# ---------------------------------------------------------------- hamiltonian

def interaction_matrix(positions, c6):
    """U_ij = C / |r_i - r_j|^6 (hamiltonian.py:66). Coincident atoms raise."""
    pos = np.asarray(positions, dtype=float)
    n = len(pos)
    u = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            d2 = float(((pos[i] - pos[j]) ** 2).sum())
            if d2 == 0.0:
                raise OracleError(f"atoms {i} and {j} coincide")
            u[i, j] = u[j, i] = c6 / d2 ** 3
    return u


def weighted_bit_sum(weights):
    """v[b] = sum_i w_i bit_i(b), built by index-range doubling (hamiltonian.py:83)."""
    w = np.asarray(weights, dtype=float)
    v = np.zeros(1 << len(w))
    half = 1
    for wk in w:
        v[half:2 * half] = v[:half] + wk
        half <<= 1
    return v


def interaction_diagonal(u):
    """d[b] = sum_{i<j} U_ij bit_i bit_j via the same doubling (hamiltonian.py:98)."""
    n = u.shape[0]
    d = np.zeros(1 << n)
    half = 1
    for k in range(n):
        d[half:2 * half] = d[:half] + weighted_bit_sum(u[:k, k])
        half <<= 1
    return d


def build_diagonal(deltas, u):
    """-sum delta_i n_i + sum_{i<j} U_ij n_i n_j (hamiltonian.py:114)."""
    deltas = np.asarray(deltas, dtype=float)
    if u.shape != (len(deltas), len(deltas)):
        raise OracleError("interaction matrix / detuning shape mismatch")
    return weighted_bit_sum(-deltas) + interaction_diagonal(u)


def apply_hamiltonian(omegas, diagonal, psi):
    """out[b] = d[b] psi[b] + sum_i (omega_i/2) psi[b ^ (1<<i)].

    Restates the reference's sequential numpy path (hamiltonian.py:151) which
    is bit-for-bit the same arithmetic per element as the compiled loop
    (_kernels.py:14) up to summation order.
    """
    omegas = np.asarray(omegas, dtype=float)
    n = len(omegas)
    psi = np.asarray(psi, dtype=complex)
    if psi.shape != (1 << n,):
        raise OracleError(f"state has shape {psi.shape}, expected ({1 << n},)")
    out = psi * diagonal
    src = psi.reshape((2,) * n)
    dst = out.reshape((2,) * n)
    for i in range(n):
        c = 0.5 * omegas[i]
        if c != 0.0:
            dst += c * np.flip(src, axis=n - 1 - i)
    return out


def build_dense(omegas, diagonal):
    """Dense 2^N x 2^N Hermitian matrix (hamiltonian.py:191), small N only."""
    n = len(omegas)
    if n > 14:
        raise OracleError(f"dense Hamiltonian refused for N={n} > 14")
    dim = 1 << n
    h = np.zeros((dim, dim), dtype=complex)
    rows = np.arange(dim)
    h[rows, rows] = diagonal
    for i in range(n):
        h[rows, rows ^ (1 << i)] += 0.5 * omegas[i]
    return h


# ---------------------------------------------------------------- krylov

def tridiag_exp_e1(alphas, betas, tau):
    """exp(-i tau T) e1 for the real symmetric tridiagonal T (krylov.py:54)."""
    k = len(alphas)
    if k == 1:
        return np.array([np.exp(-1j * tau * alphas[0])])
    t = np.diag(np.asarray(alphas, dtype=float))
    idx = np.arange(k - 1)
    t[idx, idx + 1] = betas
    t[idx + 1, idx] = betas
    lam, z = np.linalg.eigh(t)
    return z @ (np.exp(-1j * tau * lam) * z[0, :].conj())


def expm_multiply(matvec, psi, dt_ns, tolerance=1e-10, max_krylov_dim=100,
                  norm_epsilon=1e-14, full_reorth=True):
    """Lanczos exp(-i dt 1e-3 H) psi (krylov.py:67-125).

    Returns (out, iterations, converged, residual, alphas, betas). The
    convergence test, breakdown scale and full re-orthogonalisation follow
    krylov.py:96-117 line by line; ``full_reorth=False`` gives the plain
    three-term recurrence used by the fused GPU path (for comparison tests).
    """
    norm_in = float(np.linalg.norm(psi))
    if norm_in <= norm_epsilon:
        return np.array(psi, dtype=complex), 0, True, 0.0, [], []
    if dt_ns == 0.0:
        return np.array(psi, dtype=complex), 1, True, 0.0, [], []
    tau = dt_ns * NS_TO_US
    basis = [np.asarray(psi, dtype=complex) / norm_in]
    alphas, betas = [], []
    converged = False
    residual = math.inf
    while True:
        w = np.asarray(matvec(basis[-1]), dtype=complex)
        a = float(np.vdot(basis[-1], w).real)
        alphas.append(a)
        w = w - a * basis[-1]
        if betas:
            w = w - betas[-1] * basis[-2]
        if full_reorth:
            for v in basis:
                w = w - np.vdot(v, w) * v
        b = float(np.linalg.norm(w))
        y = tridiag_exp_e1(alphas, betas, tau)
        residual = b * abs(y[-1])
        scale = max(1.0, max(abs(x) for x in alphas), max(betas, default=0.0))
        if residual <= tolerance or b <= BREAKDOWN_RTOL * scale:
            converged = True
            break
        if len(alphas) >= max_krylov_dim:
            break
        betas.append(b)
        basis.append(w / b)
    out = np.zeros_like(basis[0])
    for coef, v in zip(y, basis):
        out += coef * v
    return out * norm_in, len(alphas), converged, float(residual), alphas, betas


# ---------------------------------------------------------------- observables

def occupations(psi):
    """<n_q> for every qubit (observables.py:82); probabilities renormalised."""
    psi = np.asarray(psi)
    n = int(round(math.log2(len(psi))))
    p = np.abs(psi) ** 2
    p = p / p.sum()
    idx = np.arange(len(psi))
    return np.array([p[((idx >> q) & 1) == 1].sum() for q in range(n)])


def correlation(psi, i, j):
    """<n_i n_j> (observables.py:102)."""
    p = np.abs(np.asarray(psi)) ** 2
    p = p / p.sum()
    idx = np.arange(len(p))
    return float((p * (((idx >> i) & 1) * ((idx >> j) & 1))).sum())


def energy(omegas, diagonal, psi):
    """<psi|H|psi> / <psi|psi> (north-star 'Energy' observable; not in rydsim)."""
    h_psi = apply_hamiltonian(omegas, diagonal, psi)
    return float(np.vdot(psi, h_psi).real / np.vdot(psi, psi).real)


def fidelity(a, b):
    """|<a|b>|^2 (observables.py:157)."""
    return float(abs(np.vdot(a, b)) ** 2)


def norm_difference(a, b):
    """||a - b||_2, global phase included (observables.py:137)."""
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)))


# ---------------------------------------------------------------- time stepping

def sample_bitstrings(psi, shots, seed):
    """Dense inverse-CDF sampling with the reference's batched PCG64 streams (observables.py:167-214)."""
    probs = np.abs(np.asarray(psi)) ** 2
    probs = probs / probs.sum()
    cdf = np.cumsum(probs)
    cdf[-1] = 1.0
    batch = 4096   # observables.py:34
    counts = [min(batch, shots - s) for s in range(0, shots, batch)]
    streams = np.random.SeedSequence(seed).spawn(len(counts))
    out = np.empty(shots, dtype=np.int64)
    pos = 0
    for count, stream in zip(counts, streams):
        rng = np.random.Generator(np.random.PCG64(stream))
        out[pos:pos + count] = np.searchsorted(cdf, rng.random(count), side="right")
        pos += count
    return out


def memory_estimate_sv(n_qubits, krylov_dim):
    """16 * 2^N * (k + 2) bytes (sv.py:45)."""
    if n_qubits < 1 or krylov_dim < 0:
        raise OracleError("need n_qubits >= 1 and krylov_dim >= 0")
    return 16 * (1 << n_qubits) * (krylov_dim + 2)


def evolve_sv(omegas, deltas, dt_ns, u, tolerance=1e-10, max_krylov_dim=100,
              initial=None, observe_every=1, full_reorth=True, with_energy=False):
    """Exact piecewise-constant evolution (sv.py:80-162).

    ``omegas``/``deltas`` have shape (K, N) (DiscretizedSequence, pulses.py:266).
    The interaction diagonal is assembled once and the detuning part per step
    exactly as sv.py:116 and sv.py:127-129 do. Returns a dict with the final
    state, per-step Krylov iterations/residuals and occupation records
    (every ``observe_every`` applied steps, 1-based; 0 = final only,
    observables.py:246). ``with_energy`` adds <psi_{k+1}|H_k|psi_{k+1}>.
    """
    omegas = np.asarray(omegas, dtype=float)
    deltas = np.asarray(deltas, dtype=float)
    k_steps, n = omegas.shape
    dim = 1 << n
    if initial is None:
        psi = np.zeros(dim, dtype=complex)
        psi[0] = 1.0
    else:
        psi = np.array(initial, dtype=complex)
    diag_int = interaction_diagonal(u)
    iters, resid, records, energies = [], [], [], []
    for k in range(k_steps):
        diag = diag_int + weighted_bit_sum(-deltas[k])
        mv = lambda v, d=diag, om=omegas[k]: apply_hamiltonian(om, d, v)
        psi, it, conv, res, _, _ = expm_multiply(
            mv, psi, float(dt_ns), tolerance, max_krylov_dim, full_reorth=full_reorth)
        if not conv:
            raise OracleError(f"Krylov did not converge at step {k} (residual {res:.3e})")
        iters.append(it)
        resid.append(res)
        step = k + 1
        due = (step == k_steps) if observe_every == 0 else (step % observe_every == 0)
        if due:
            records.append((step, step * dt_ns, occupations(psi)))
            if with_energy:
                energies.append((step, energy(omegas[k], diag, psi)))
    return {"final_state": psi, "iterations": iters, "residuals": resid,
            "occupations": records, "energies": energies}


def evolve_dense(omegas, deltas, dt_ns, u, initial=None):
    """Dense eigendecomposition evolution (oracle.py:42), N <= 12."""
    omegas = np.asarray(omegas, dtype=float)
    deltas = np.asarray(deltas, dtype=float)
    k_steps, n = omegas.shape
    if n > 12:
        raise OracleError(f"oracle backend refuses N={n} > 12")
    psi = np.zeros(1 << n, dtype=complex)
    if initial is None:
        psi[0] = 1.0
    else:
        psi[:] = initial
    cache = None
    for k in range(k_steps):
        key = (omegas[k].tobytes(), deltas[k].tobytes())
        if cache is None or cache[0] != key:
            h = build_dense(omegas[k], build_diagonal(deltas[k], u))
            lam, z = np.linalg.eigh(h)
            cache = (key, lam, z)
        _, lam, z = cache
        psi = z @ (np.exp(-1j * dt_ns * NS_TO_US * lam) * (z.conj().T @ psi))
    return psi


# ---------------------------------------------------------------- pulses

def blackman_window(n):
    """Three-term Blackman window with exact-zero edges (pulses.py:37)."""
    if n < 1:
        raise OracleError("window length must be >= 1")
    if n == 1:
        return np.zeros(1)
    x = 2.0 * np.pi * np.arange(n) / (n - 1)
    w = 0.42 - 0.5 * np.cos(x) + 0.08 * np.cos(2.0 * x)
    w[0] = w[-1] = 0.0
    return w


def sample_segment(seg):
    """1 ns samples of one segment tuple (pulses.py:76-150).

    ('constant', dur, value) | ('ramp', dur, start, stop) |
    ('blackman', dur, area) | ('spline', dur, points)
    """
    kind, dur = seg[0], int(seg[1])
    if kind == "constant":
        return np.full(dur, float(seg[2]))
    if kind == "ramp":
        return np.linspace(float(seg[2]), float(seg[3]), dur)
    if kind == "blackman":
        area = float(seg[2])
        if area == 0.0:
            return np.zeros(dur)
        w = blackman_window(dur)
        return w * (area / w.sum())
    if kind == "spline":
        pts = seg[2]
        t = np.array([p[0] for p in pts], dtype=float)
        v = np.array([p[1] for p in pts], dtype=float)
        if len(pts) == 2:
            return np.interp(np.arange(dur), t, v)
        return CubicSpline(t, v, bc_type="natural")(np.arange(dur))
    raise OracleError(f"unknown segment kind {kind!r}")


def sample_channels(channels, duration_ns):
    """(N, T) samples, zero padded (pulses.py:158, pulses.py:244)."""
    out = np.zeros((len(channels), duration_ns))
    for q, segs in enumerate(channels):
        parts = [sample_segment(s) for s in segs]
        row = np.concatenate(parts) if parts else np.zeros(0)
        if len(row) > duration_ns:
            raise OracleError(f"qubit {q}: channel overruns the program")
        out[q, :len(row)] = row
    return out


def discretize(samples, dt_ns):
    """Midpoint rule (x[floor m] + x[min(ceil m, T-1)])/2, m=(n+1/2)dt (pulses.py:286-315).

    ``samples`` has shape (N, T); returns (K, N).
    """
    t = samples.shape[1]
    if dt_ns < 1 or t % dt_ns:
        raise OracleError(f"duration {t} not divisible by dt={dt_ns}")
    m = (np.arange(t // dt_ns) + 0.5) * dt_ns
    lo = np.floor(m).astype(int)
    hi = np.minimum(np.ceil(m).astype(int), t - 1)
    return 0.5 * (samples[:, lo] + samples[:, hi]).T


# ---------------------------------------------------------------- generators

def chain_positions(n, spacing_um=DEFAULT_SPACING_UM):
    """generator.py:28."""
    return [(i * spacing_um, 0.0) for i in range(n)]


def grid_positions(rows, cols, spacing_um=DEFAULT_SPACING_UM):
    """generator.py:38 (row-major, x = column)."""
    return [(c * spacing_um, r * spacing_um) for r in range(rows) for c in range(cols)]


def ring_positions(n, spacing_um=DEFAULT_SPACING_UM):
    """Regular polygon with nearest-neighbour distance ``spacing_um`` (config[0] register)."""
    radius = spacing_um / (2.0 * math.sin(math.pi / n))
    return [(radius * math.cos(2 * math.pi * i / n), radius * math.sin(2 * math.pi * i / n))
            for i in range(n)]


def adiabatic_channels(n, duration_ns=1000, omega_peak=TWO_PI,
                       delta_start=-3 * TWO_PI, delta_end=2 * TWO_PI):
    """Global Blackman drive + linear detuning sweep (generator.py:50)."""
    w = blackman_window(duration_ns)
    area = omega_peak * w.sum() / w.max()
    omega = [[("blackman", duration_ns, area)] for _ in range(n)]
    delta = [[("ramp", duration_ns, delta_start, delta_end)] for _ in range(n)]
    return omega, delta


def random_channels(rng, n, duration_ns, segments=3, omega_scale=2 * TWO_PI,
                    delta_scale=2 * TWO_PI):
    """Random constant/ramp channels, same RNG draw order as generator.py:73."""
    edges = np.sort(rng.choice(np.arange(1, duration_ns), segments - 1, replace=False))
    lengths = np.diff(np.concatenate([[0], edges, [duration_ns]])).astype(int)

    def channel(scale, signed):
        lo = -scale if signed else 0.0
        segs = []
        for length in lengths:
            if rng.random() < 0.5:
                segs.append(("constant", int(length), rng.uniform(lo, scale)))
            else:
                segs.append(("ramp", int(length), rng.uniform(lo, scale), rng.uniform(lo, scale)))
        return segs

    omega = [channel(omega_scale, False) for _ in range(n)]
    delta = [channel(delta_scale, True) for _ in range(n)]
    return omega, delta
