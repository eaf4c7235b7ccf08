"""Generate golden vectors by running the REAL reference (rydsim) in the build container.

Usage (build container only -- /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``. The fixtures are committed; tests only read them.
Each case records the reference call it came from so the parity tests can
replay the same inputs through the oracle restatement and through the CUDA path.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from rydsim.generator import adiabatic_program, chain_register, grid_register, random_program  # noqa: E402
from rydsim.hamiltonian import (  # noqa: E402
    HamiltonianSlice, Register, apply_hamiltonian, build_diagonal, interaction_matrix)
from rydsim.krylov import KrylovConfig, expm_multiply  # noqa: E402
from rydsim.observables import ObservableSpec, correlation, occupations  # noqa: E402
from rydsim.pulses import ChannelProgram, Constant, Ramp, discretize, sample_program  # noqa: E402
from rydsim.sequence_io import parse_sequence  # noqa: E402
from rydsim.sv import SvRunConfig, evolve_sv  # noqa: E402

TWO_PI = 2 * math.pi


def random_slice(rng, n):
    # same draws as the reference test helper (tests/test_hamiltonian.py:48)
    omegas = rng.uniform(0.0, 4.0, n)
    deltas = rng.uniform(-3.0, 3.0, n)
    u = rng.uniform(0.0, 2.0, (n, n))
    u = np.triu(u, 1)
    return omegas, deltas, u + u.T


def ring_positions(n, spacing):
    r = spacing / (2.0 * math.sin(math.pi / n))
    return tuple((r * math.cos(2 * math.pi * i / n), r * math.sin(2 * math.pi * i / n))
                 for i in range(n))


def gen_apply():
    out = {}
    for n in (1, 2, 3, 4, 5, 7, 8, 10, 11, 12, 13):
        rng = np.random.default_rng(1000 + n)
        om, de, u = random_slice(rng, n)
        s = HamiltonianSlice.from_parameters(om, de, u)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        out[f"n{n}_omegas"] = om
        out[f"n{n}_deltas"] = de
        out[f"n{n}_u"] = u
        out[f"n{n}_psi"] = psi
        out[f"n{n}_diag"] = s.diagonal
        out[f"n{n}_hpsi"] = apply_hamiltonian(s, psi)
    np.savez_compressed(os.path.join(HERE, "apply_hamiltonian.npz"), **out)


def gen_expm():
    out = {}
    for n in range(2, 11):
        rng = np.random.default_rng(2000 + n)
        om, de, u = random_slice(rng, n)
        s = HamiltonianSlice.from_parameters(om, de, u)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        psi /= np.linalg.norm(psi)
        dt = 10.0 * (1 + n % 3)
        res, rep = expm_multiply(lambda v: apply_hamiltonian(s, v), psi, dt, KrylovConfig(1e-10))
        out[f"n{n}_omegas"] = om
        out[f"n{n}_deltas"] = de
        out[f"n{n}_u"] = u
        out[f"n{n}_psi"] = psi
        out[f"n{n}_dt"] = np.array(dt)
        out[f"n{n}_out"] = res
        out[f"n{n}_iterations"] = np.array(rep.iterations)
    np.savez_compressed(os.path.join(HERE, "expm_multiply.npz"), **out)


def run_case(name, reg, prog, dt, tol=1e-10, every=1, pairs=()):
    seq = discretize(sample_program(prog), dt)
    specs = [ObservableSpec("occupation", (), every_n_steps=every)]
    if pairs:
        specs.append(ObservableSpec("correlation", tuple(q for p in pairs for q in p),
                                    every_n_steps=0))
    res = evolve_sv(seq, reg, SvRunConfig(krylov=KrylovConfig(tol), observables=tuple(specs)))
    occ = np.array([r.values for r in res.observables if r.kind == "occupation"])
    occ_t = np.array([r.t_ns for r in res.observables if r.kind == "occupation"])
    d = {
        "positions": np.array(reg.positions_um),
        "c6": np.array(reg.interaction_c),
        "omegas": seq.omegas, "deltas": seq.deltas, "dt": np.array(dt),
        "tol": np.array(tol), "every": np.array(every),
        "occ": occ, "occ_t": occ_t,
        "iterations": np.array([r.iterations for r in res.krylov_reports]),
        "u": interaction_matrix(reg),
    }
    n = reg.qubit_count
    psi = res.final_state
    if n <= 14:
        d["final_state"] = psi
    else:
        # large registers: size-independent checksums of the final state
        rng = np.random.default_rng(77)
        probe = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        d["probe_overlap"] = np.array(np.vdot(probe, psi))
        d["norm"] = np.array(np.linalg.norm(psi))
        d["amp_head"] = psi[:64].copy()
    if pairs:
        d["pairs"] = np.array(pairs)
        d["corr"] = np.array([r.values for r in res.observables if r.kind == "correlation"][-1])
    # energy of the final state w.r.t. the last slice (north-star observable)
    last = HamiltonianSlice.from_parameters(seq.omegas[-1], seq.deltas[-1], interaction_matrix(reg))
    d["energy_last"] = np.array(np.vdot(psi, apply_hamiltonian(last, psi)).real)
    np.savez_compressed(os.path.join(HERE, f"evolve_{name}.npz"), **d)
    print(name, "steps", seq.step_count, "max iters", d["iterations"].max())


def gen_evolve():
    # configs[0]: N=10 ring, constant Omega = 2pi rad/us, delta = 0, 1 us, Occupation (+Energy)
    n = 10
    reg = Register(ring_positions(n, 7.0), 5_000_000.0)
    prog = ChannelProgram.from_channels([[Constant(1000, TWO_PI)] for _ in range(n)],
                                        [[Constant(1000, 0.0)] for _ in range(n)], 1000)
    run_case("ring10", reg, prog, 10, pairs=((0, 1), (0, 5), (3, 4)))

    # reference test workloads (tests/test_sv.py)
    reg, prog = adiabatic_program(5, duration_ns=400)
    run_case("adiabatic5", reg, prog, 10)
    reg, prog = adiabatic_program(9, duration_ns=300)
    run_case("adiabatic9", reg, prog, 10, every=10, pairs=((0, 1), (4, 8)))
    rng = np.random.default_rng(0)
    for trial in range(3):
        n = int(rng.integers(2, 7))
        reg = chain_register(n, spacing_um=9.0)
        prog = random_program(rng, n, duration_ns=40)
        run_case(f"random{trial}", reg, prog, 4, tol=1e-12)
    reg = Register(((0.0, 0.0), (3.0, 0.0)), 5e6)
    prog = ChannelProgram.from_channels([[Constant(500, TWO_PI)]] * 2, [[Constant(500, 0.0)]] * 2, 500)
    run_case("blockade2", reg, prog, 1, tol=1e-12, every=50)

    # per-atom detuning map on a random 2D register (configs[3] shape, small N)
    rng = np.random.default_rng(11)
    n = 12
    pos = []
    while len(pos) < n:
        p = rng.uniform(0, 30.0, 2)
        if all(np.hypot(*(p - q)) >= 5.0 for q in pos):
            pos.append(p)
    reg = Register(tuple(map(tuple, pos)), 5_420_000.0)
    dmap = rng.uniform(0.5, 1.0, n)
    prog = ChannelProgram.from_channels(
        [[Constant(200, 1.5 * TWO_PI)] for _ in range(n)],
        [[Ramp(200, -6.0 * dmap[q], 6.0 * dmap[q])] for q in range(n)], 200)
    run_case("detmap12", reg, prog, 10, every=5, pairs=((0, 1), (2, 7)))

    # configs[1]: N=20 4x5 lattice, 5.6 um, delta sweep -6 -> +6 rad/us over 3 us.
    # Only the first 100 ns (10 steps) of the sweep: enough to pin the large-N path.
    reg = grid_register(4, 5, spacing_um=5.6, interaction_c=5_420_000.0)
    prog = ChannelProgram.from_channels(
        [[Constant(3000, TWO_PI)] for _ in range(20)],
        [[Ramp(3000, -6.0, 6.0)] for _ in range(20)], 3000)
    seq_full = sample_program(prog)
    from rydsim.pulses import SampledSequence
    head = SampledSequence(seq_full.omega[:, :100].copy(), seq_full.delta[:, :100].copy())
    seq = discretize(head, 10)
    res = evolve_sv(seq, reg, SvRunConfig(krylov=KrylovConfig(1e-10),
                                          observables=(ObservableSpec("occupation", (), 1),)))
    psi = res.final_state
    rng = np.random.default_rng(77)
    probe = rng.standard_normal(2 ** 20) + 1j * rng.standard_normal(2 ** 20)
    np.savez_compressed(
        os.path.join(HERE, "evolve_lattice20.npz"),
        positions=np.array(reg.positions_um), c6=np.array(reg.interaction_c),
        omegas=seq.omegas, deltas=seq.deltas, dt=np.array(10), tol=np.array(1e-10),
        every=np.array(1),
        occ=np.array([r.values for r in res.observables]),
        occ_t=np.array([r.t_ns for r in res.observables]),
        iterations=np.array([r.iterations for r in res.krylov_reports]),
        u=interaction_matrix(reg),
        probe_overlap=np.array(np.vdot(probe, psi)), norm=np.array(np.linalg.norm(psi)),
        amp_head=psi[:64].copy())
    print("lattice20 iters", [r.iterations for r in res.krylov_reports])


def gen_pulses():
    out = {}
    reg, prog = adiabatic_program(3, duration_ns=120)
    s = sample_program(prog)
    out["adiabatic_omega"] = s.omega
    out["adiabatic_delta"] = s.delta
    out["adiabatic_disc_omega_dt8"] = discretize(s, 8).omegas
    out["adiabatic_disc_delta_dt8"] = discretize(s, 8).deltas
    rng = np.random.default_rng(5)
    prog = random_program(rng, 3, duration_ns=60)
    s = sample_program(prog)
    out["random_omega"] = s.omega
    out["random_delta"] = s.delta
    out["random_disc_omega_dt1"] = discretize(s, 1).omegas
    # shipped example sequences
    for name in ("sequence_blockade_2q", "sequence_adiabatic_5q"):
        reg, prog = parse_sequence(f"/root/reference/pkg/configs/{name}.json")
        s = sample_program(prog)
        out[f"{name}_omega"] = s.omega
        out[f"{name}_delta"] = s.delta
        out[f"{name}_u"] = interaction_matrix(reg)
    np.savez_compressed(os.path.join(HERE, "pulses.npz"), **out)


def gen_diag_checks():
    out = {}
    for n in (1, 2, 6, 9):
        rng = np.random.default_rng(300 + n)
        _, de, u = random_slice(rng, n)
        out[f"n{n}_deltas"] = de
        out[f"n{n}_u"] = u
        out[f"n{n}_diag"] = build_diagonal(de, u)
    reg = Register(((0.0, 0.0), (5.0, 0.0), (10.0, 0.0)), 5_000_000.0)
    out["line3_u"] = interaction_matrix(reg)
    np.savez_compressed(os.path.join(HERE, "diagonal.npz"), **out)


def gen_sampling():
    """rydsim.observables.sample_bitstrings on random normalised states (dense inverse-CDF path)."""
    from rydsim.observables import sample_bitstrings

    out = {}
    for n, shots, seed in ((1, 50, 1), (5, 1000, 7), (10, 5000, 2025), (14, 9000, 3)):
        rng = np.random.default_rng(400 + n)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        if n == 10:   # a peaked state: most of the weight on a few indices
            psi[rng.integers(0, 2 ** n, 3)] *= 40.0
        psi /= np.linalg.norm(psi)
        out[f"n{n}_psi"] = psi
        out[f"n{n}_shots"] = shots
        out[f"n{n}_seed"] = seed
        out[f"n{n}_idx"] = sample_bitstrings(psi, shots, seed)
    np.savez_compressed(os.path.join(HERE, "sampling.npz"), **out)


def _segment_doc(seg):
    d = {"kind": type(seg).__name__, "duration_ns": seg.duration_ns}
    for k in ("value", "start", "stop", "area", "points"):
        if hasattr(seg, k):
            v = getattr(seg, k)
            d[k] = [list(p) for p in v] if k == "points" else v
    return d


def gen_runs():
    """rydsim.runner.execute_run (backend sv) on the reference's own sequence/config fixtures and on a
    variant with correlations, snapshots, an initial bitstring and samples. The inputs are stored as a
    plain program description (register + segments) that the tests rebuild with the mirror's types."""
    from rydsim.observables import ObservableSpec as RefSpec
    from rydsim.runner import execute_run
    from rydsim.sequence_io import parse_config, parse_sequence

    cfg_dir = "/root/reference/pkg/configs"
    reg, prog = parse_sequence(os.path.join(cfg_dir, "sequence_adiabatic_5q.json"))
    base = parse_config(os.path.join(cfg_dir, "run_sv.json"))
    import dataclasses

    variants = {
        "adiabatic5": base,
        "adiabatic5_var": dataclasses.replace(
            base, dt_ns=20, initial_bits=0b00100, seed=11, sample_shots=3000, snapshot_every=10,
            observables=(RefSpec("occupation", (0, 2, 4), 5), RefSpec("correlation", (0, 1, 1, 3), 0))),
    }
    out = {}
    for name, cfg in variants.items():
        doc = execute_run(reg, prog, cfg).strip_volatile()
        out[name] = {"document": doc,
                     "register": {"positions_um": [list(p) for p in reg.positions_um],
                                  "interaction_c": reg.interaction_c},
                     "program": {"duration_ns": prog.duration_ns,
                                 "omega": [[_segment_doc(s) for s in ch] for ch in prog.omega],
                                 "delta": [[_segment_doc(s) for s in ch] for ch in prog.delta]},
                     "config": {"dt_ns": cfg.dt_ns, "initial_bits": cfg.initial_bits, "seed": cfg.seed,
                                "sample_shots": cfg.sample_shots, "snapshot_every": cfg.snapshot_every,
                                "tolerance": cfg.krylov.tolerance, "max_krylov_dim": cfg.krylov.max_krylov_dim,
                                "observables": [[s.kind, list(s.qubits), s.every_n_steps]
                                                for s in cfg.observables]}}
    with open(os.path.join(HERE, "runs_sv.json"), "w") as fh:
        json.dump(out, fh)


def gen_lattice20_full():
    """configs[1] for its whole length: N=20 4x5 lattice, 5.6 um, delta sweep -6 -> +6 rad/us over
    3 us (300 steps of 10 ns), occupations every 10 steps, energy at the end."""
    reg = grid_register(4, 5, spacing_um=5.6, interaction_c=5_420_000.0)
    prog = ChannelProgram.from_channels(
        [[Constant(3000, TWO_PI)] for _ in range(20)],
        [[Ramp(3000, -6.0, 6.0)] for _ in range(20)], 3000)
    seq = discretize(sample_program(prog), 10)
    res = evolve_sv(seq, reg, SvRunConfig(krylov=KrylovConfig(1e-10),
                                          observables=(ObservableSpec("occupation", (), 10),)))
    psi = res.final_state
    rng = np.random.default_rng(77)
    probe = rng.standard_normal(2 ** 20) + 1j * rng.standard_normal(2 ** 20)
    occ = [r for r in res.observables if r.kind == "occupation"]
    last = HamiltonianSlice.from_parameters(seq.omegas[-1], seq.deltas[-1], interaction_matrix(reg))
    np.savez_compressed(
        os.path.join(HERE, "evolve_lattice20_full.npz"),
        positions=np.array(reg.positions_um), c6=np.array(reg.interaction_c),
        omegas=seq.omegas, deltas=seq.deltas, dt=np.array(10), tol=np.array(1e-10),
        every=np.array(10),
        occ=np.array([r.values for r in occ]), occ_t=np.array([r.t_ns for r in occ]),
        energy_last=np.array(np.vdot(psi, apply_hamiltonian(last, psi)).real),
        iterations=np.array([r.iterations for r in res.krylov_reports]),
        probe_overlap=np.array(np.vdot(probe, psi)), norm=np.array(np.linalg.norm(psi)),
        amp_head=psi[:64].copy(), amp_tail=psi[-64:].copy())
    print("lattice20 full: steps", seq.step_count, "iters max", res.max_krylov_iterations)


if __name__ == "__main__":
    if "--lattice20-full" in sys.argv:   # configs[1] full-length fixture (minutes of CPU)
        gen_lattice20_full()
        sys.exit(0)
    if "--sampling" in sys.argv:   # regenerate only the sampling fixture
        gen_sampling()
        sys.exit(0)
    if "--runs" in sys.argv:       # regenerate only the run-document fixture
        gen_runs()
        sys.exit(0)
    gen_runs()
    gen_sampling()
    gen_apply()
    gen_expm()
    gen_diag_checks()
    gen_pulses()
    gen_evolve()
    with open(os.path.join(HERE, "PROVENANCE.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "rydsim 0.1.0 from /root/reference/pkg/src",
                   "numpy": np.__version__}, fh, indent=1)
