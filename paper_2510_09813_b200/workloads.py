"""Synthetic registers and pulses for the BASELINE.json configurations (no datasets needed).

configs[0]  ring10     N=10 ring, constant Omega = 2pi rad/us, delta = 0, 1 us
configs[1]  lattice20  N=20 4x5 lattice, 5.6 um, delta sweep -6 -> +6 rad/us over 3 us
configs[2]  lattice27  N=27 3x9 lattice global pulse (Blackman drive + linear sweep)
configs[3]  random29   N=29 random 2D register with a per-atom detuning map, 1 us
configs[4]  random33   N=33 random 2D register, 1 us (sharded configuration)

Interaction constant C6 = 2pi * 862690 rad um^6/us (Rb 70S), the magnitude the
reference's example configs use (generator.py:23 ships 5e6).
"""

from __future__ import annotations

import math

import numpy as np

from .hamiltonian import Register
from .pulses import Blackman, ChannelProgram, Constant, Ramp, blackman_window, discretize, sample_program

C6_RB70 = 2 * math.pi * 862690.0
TWO_PI = 2 * math.pi


def random_register(n: int, seed: int = 2025, mean_spacing_um: float = 7.0, min_dist_um: float = 6.0,
                    c6: float = C6_RB70):
    """Uniform positions in a square of side mean_spacing * sqrt(n), rejection-sampled to min_dist."""
    rng = np.random.default_rng(seed)
    side = mean_spacing_um * math.sqrt(n)
    pos = []
    while len(pos) < n:
        p = rng.uniform(0.0, side, 2)
        if all(math.hypot(p[0] - q[0], p[1] - q[1]) >= min_dist_um for q in pos):
            pos.append((float(p[0]), float(p[1])))
    detuning_map = rng.uniform(0.6, 1.0, n)
    return Register(tuple(pos), c6), detuning_map


def grid_register(rows, cols, spacing_um, c6=C6_RB70):
    return Register(tuple((c * spacing_um, r * spacing_um) for r in range(rows) for c in range(cols)), c6)


def ring_register(n, spacing_um=7.0, c6=5_000_000.0):
    r = spacing_um / (2.0 * math.sin(math.pi / n))
    return Register(tuple((r * math.cos(2 * math.pi * i / n), r * math.sin(2 * math.pi * i / n))
                          for i in range(n)), c6)


def sweep_program(n, duration_ns, omega_peak, delta_start, delta_stop, detuning_map=None, blackman=True):
    dmap = np.ones(n) if detuning_map is None else np.asarray(detuning_map)
    if blackman:
        w = blackman_window(duration_ns)
        area = omega_peak * w.sum() / w.max()
        omega = [[Blackman(duration_ns, area)] for _ in range(n)]
    else:
        omega = [[Constant(duration_ns, omega_peak)] for _ in range(n)]
    delta = [[Ramp(duration_ns, delta_start * dmap[q], delta_stop * dmap[q])] for q in range(n)]
    return ChannelProgram.from_channels(omega, delta, duration_ns)


def config(name: str, dt_ns: int = 10, n_override=None):
    """(register, DiscretizedSequence, description) for a BASELINE.json configuration."""
    if name == "ring10":
        n = 10
        reg = ring_register(n)
        prog = ChannelProgram.from_channels([[Constant(1000, TWO_PI)] for _ in range(n)],
                                            [[Constant(1000, 0.0)] for _ in range(n)], 1000)
    elif name == "lattice20":
        reg = grid_register(4, 5, 5.6)
        prog = sweep_program(20, 3000, TWO_PI, -6.0, 6.0, blackman=False)
    elif name == "lattice27":
        reg = grid_register(3, 9, 6.5)
        prog = sweep_program(27, 1000, 1.5 * TWO_PI, -6.0, 6.0)
    elif name in ("random29", "random33"):
        n = n_override or (29 if name == "random29" else 33)
        reg, dmap = random_register(n)
        prog = sweep_program(n, 1000, 1.5 * TWO_PI, -6.0, 6.0, detuning_map=dmap)
    else:
        raise ValueError(f"unknown config {name!r}")
    seq = discretize(sample_program(prog), dt_ns)
    return reg, seq
