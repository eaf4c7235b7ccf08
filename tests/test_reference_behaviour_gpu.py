"""The reference's behavioural tests for the state-vector path (tests/test_sv.py, test_krylov.py,
test_observables.py sampling section), restated against the B200 path through the public API:
physical limits (Rabi phase, blockade, norm), exactness properties (constant pulse in one step,
scaling, backward evolution), reporting (snapshots, wall times, non-convergence reported, memory
refusal) and the sampler's statistics. Tolerances as in the reference tests."""

import math

import numpy as np
import pytest

from oracle import sv_oracle as O

pytestmark = pytest.mark.gpu
TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def rs():
    import paper_2510_09813_b200 as pkg

    return pkg


def constant_seq(rs, n, omega, delta, duration, dt):
    k = duration // dt
    return rs.DiscretizedSequence(dt, np.full((k, n), float(omega)), np.full((k, n), float(delta)), duration)


def far_register(rs, n):
    return rs.Register(tuple((1e6 * i, 0.0) for i in range(n)), 5e6)


def chain(rs, n, spacing):
    return rs.Register(tuple((spacing * i, 0.0) for i in range(n)), 5e6)


def host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def random_slice(rng, n):
    om = rng.uniform(0.0, 4.0, n)
    de = rng.uniform(-3.0, 3.0, n)
    u = np.triu(rng.uniform(0.0, 2.0, (n, n)), 1)
    return om, de, u + u.T


class TestEvolve:
    def test_zero_pulse_identity(self, rs):
        res = rs.evolve_sv(constant_seq(rs, 3, 0.0, 0.0, 100, 10), far_register(rs, 3))
        expected = np.zeros(8, complex)
        expected[0] = 1.0
        assert np.abs(host(res.final_state) - expected).max() <= 1e-15

    def test_blockade_suppression(self, rs):
        # resonant pi pulse on two atoms deep inside the blockade radius: |11> stays empty
        reg = rs.Register(((0.0, 0.0), (3.0, 0.0)), 5e6)
        res = rs.evolve_sv(constant_seq(rs, 2, TWO_PI, 0.0, 500, 1), reg,
                           rs.SvRunConfig(krylov=rs.KrylovConfig(1e-12)))
        assert abs(host(res.final_state)[3]) ** 2 <= 0.01

    def test_norm_conservation(self, rs):
        # adiabatic sweep (generator.py:50 shape: global Blackman drive, linear detuning ramp)
        from paper_2510_09813_b200.pulses import blackman_window

        w = blackman_window(400)
        area = TWO_PI * w.sum() / w.max()
        prog = rs.ChannelProgram.from_channels([[rs.Blackman(400, area)] for _ in range(5)],
                                               [[rs.Ramp(400, -3 * TWO_PI, 2 * TWO_PI)] for _ in range(5)], 400)
        seq = rs.discretize(rs.sample_program(prog), 10)
        res = rs.evolve_sv(seq, chain(rs, 5, 7.0), rs.SvRunConfig(krylov=rs.KrylovConfig(1e-10)))
        assert abs(np.linalg.norm(host(res.final_state)) - 1.0) <= 10 * 1e-10 * 40

    def test_constant_pulse_single_step_exact(self, rs):
        n, duration, p = 3, 240, 1e-12
        reg = chain(rs, n, 8.0)
        fine = rs.evolve_sv(constant_seq(rs, n, 1.7, -0.9, duration, 1), reg, rs.SvRunConfig(krylov=rs.KrylovConfig(p)))
        single = rs.evolve_sv(constant_seq(rs, n, 1.7, -0.9, duration, duration), reg,
                              rs.SvRunConfig(krylov=rs.KrylovConfig(p)))
        assert rs.norm_difference(fine.final_state, single.final_state) <= 100 * p

    def test_snapshots_and_wall_times(self, rs):
        res = rs.evolve_sv(constant_seq(rs, 2, 1.0, 0.0, 100, 10), far_register(rs, 2), rs.SvRunConfig(snapshot_every=5))
        assert [t for t, _ in res.snapshots] == [50.0, 100.0]
        assert len(res.step_wall_times_s) == 10

    def test_initial_state_override(self, rs):
        plus = np.array([1.0, 1.0], complex) / math.sqrt(2)
        res = rs.evolve_sv(constant_seq(rs, 1, 0.0, TWO_PI, 10, 10), far_register(rs, 1),
                           rs.SvRunConfig(initial_state=plus))
        expected = np.array([1.0, np.exp(1j * TWO_PI * 0.01)]) / math.sqrt(2)   # detuning adds +delta t
        assert rs.norm_difference(res.final_state, expected) <= 1e-10

    def test_qubit_cap_override(self, rs):
        res = rs.evolve_sv(constant_seq(rs, 4, 1.0, 0.0, 10, 10), far_register(rs, 4),
                           rs.SvRunConfig(qubit_cap=3, allow_above_cap=True))
        assert tuple(res.final_state.shape) == (16,)

    def test_memory_budget_refusal(self, rs):
        with pytest.raises(rs.MemoryBudgetError) as err:
            rs.evolve_sv(constant_seq(rs, 20, 1.0, 0.0, 10, 10), far_register(rs, 20),
                         rs.SvRunConfig(memory_budget_bytes=10 ** 6))
        assert err.value.required_bytes == rs.memory_estimate_sv(20, 15)


class TestExpm:
    def test_norm_preservation(self, rs):
        rng = np.random.default_rng(77)
        s = rs.HamiltonianSlice.from_parameters(*random_slice(rng, 8))
        psi = rng.standard_normal(256) + 1j * rng.standard_normal(256)
        out, _ = rs.expm_multiply(s, psi, 50.0, rs.KrylovConfig(1e-8))
        assert abs(np.linalg.norm(out) - np.linalg.norm(psi)) <= 10 * 1e-8

    def test_tolerance_monotonicity(self, rs):
        rng = np.random.default_rng(5)
        s = rs.HamiltonianSlice.from_parameters(*random_slice(rng, 8))
        psi = rng.standard_normal(256) + 1j * rng.standard_normal(256)
        iters = [rs.expm_multiply(s, psi, 20.0, rs.KrylovConfig(p))[1].iterations
                 for p in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12)]
        assert all(a <= b for a, b in zip(iters, iters[1:]))

    def test_scaling_invariance(self, rs):
        rng = np.random.default_rng(13)
        s = rs.HamiltonianSlice.from_parameters(*random_slice(rng, 6))
        psi = rng.standard_normal(64) + 1j * rng.standard_normal(64)
        a = 2.7 - 0.4j
        out1, _ = rs.expm_multiply(s, a * psi, 15.0, rs.KrylovConfig(1e-10))
        out2, _ = rs.expm_multiply(s, psi, 15.0, rs.KrylovConfig(1e-10))
        assert np.linalg.norm(out1 - a * out2) <= 1e-12 * np.linalg.norm(out1)

    def test_non_convergence_reported_not_raised(self, rs):
        rng = np.random.default_rng(1)
        n = 9
        s = rs.HamiltonianSlice.from_parameters(rng.uniform(100.0, 200.0, n), rng.uniform(-3000.0, 3000.0, n),
                                                np.zeros((n, n)))
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        _, rep = rs.expm_multiply(s, psi, 1000.0, rs.KrylovConfig(tolerance=1e-12, max_krylov_dim=5))
        assert not rep.converged and rep.iterations == 5 and rep.residual > 1e-12

    def test_iterations_bounded(self, rs):
        rng = np.random.default_rng(17)
        s = rs.HamiltonianSlice.from_parameters(*random_slice(rng, 7))
        psi = rng.standard_normal(128) + 1j * rng.standard_normal(128)
        _, rep = rs.expm_multiply(s, psi, 100.0, rs.KrylovConfig(tolerance=1e-12, max_krylov_dim=40))
        assert rep.iterations <= 40


class TestSampling:
    def test_ground_state(self, rs):
        psi = np.zeros(32, complex)
        psi[0] = 1.0
        assert np.all(rs.sample_bitstrings(psi, 100, 1) == 0)

    def test_equal_superposition_frequency(self, rs):
        out = rs.sample_bitstrings(np.array([1.0, 1.0], complex) / math.sqrt(2), 100_000, 2)
        assert 0.494 <= np.mean(out == 1) <= 0.506   # 4 sigma around 1/2

    def test_deterministic(self, rs):
        rng = np.random.default_rng(8)
        psi = rng.standard_normal(16) + 1j * rng.standard_normal(16)
        psi /= np.linalg.norm(psi)
        a = rs.sample_bitstrings(psi, 10_000, 99)
        assert np.array_equal(a, rs.sample_bitstrings(psi, 10_000, 99))
        assert np.array_equal(a, O.sample_bitstrings(psi, 10_000, 99))


class TestDiscretizationOrder:
    def test_second_order_in_dt(self, rs):
        # reference tests/test_sv.py:145-159: adiabatic_program(2, 320 ns) on the default chain
        # (generator.py:28,50: 7 um spacing, C = 5e6, Blackman drive, -3*2pi -> 2*2pi sweep);
        # halving dt cuts the final-state error ~4x (midpoint sampling, pulses.py discretize)
        reg = rs.Register(tuple((7.0 * i, 0.0) for i in range(2)), 5_000_000.0)
        w = rs.pulses.blackman_window(320)
        area = TWO_PI * w.sum() / w.max()
        prog = rs.ChannelProgram.from_channels([[rs.Blackman(320, area)] for _ in range(2)],
                                               [[rs.Ramp(320, -3 * TWO_PI, 2 * TWO_PI)] for _ in range(2)], 320)
        sampled = rs.sample_program(prog)
        cfg = rs.SvRunConfig(krylov=rs.KrylovConfig(1e-12))
        ref = rs.evolve_sv(rs.discretize(sampled, 1), reg, cfg).final_state
        errors = {}
        for dt in (2, 4, 8, 16):
            out = rs.evolve_sv(rs.discretize(sampled, dt), reg, cfg).final_state
            errors[dt] = rs.norm_difference(out, ref)
        for dt in (2, 4, 8):
            ratio = errors[2 * dt] / errors[dt]
            assert 2.5 <= ratio <= 6.0, (dt, errors)


def test_snapshots_at_full_size(rs):
    # N=29: the Krylov workspace takes all of HBM, snapshots go to host memory
    from paper_2510_09813_b200 import workloads

    reg, seq = workloads.config("random29")
    sub = rs.DiscretizedSequence(seq.dt_ns, seq.omegas[:2], seq.deltas[:2], 2 * seq.dt_ns)
    res = rs.evolve_sv(sub, reg, rs.SvRunConfig(snapshot_every=1))
    assert [t for t, _ in res.snapshots] == [10.0, 20.0]
    last = res.snapshots[-1][1]
    assert isinstance(last, np.ndarray) and last.shape == (2 ** 29,)
    assert abs(np.vdot(last[:2 ** 20], last[:2 ** 20]).real) <= 1.0 + 1e-9
    # the workspace still holds all of HBM: compare on the host, then release it
    assert np.array_equal(res.final_state[: 2 ** 24].cpu().numpy(), last[: 2 ** 24])
    psi = res.release()
    assert psi.is_cuda and tuple(psi.shape) == (2 ** 29,) and res.engine is None
    assert rs.norm_difference(psi, last) == 0.0   # now there is room for other GPU work


def test_expm_multiply_at_full_size(rs):
    # one fused Lanczos step on a user-owned N=29 vector: the workspace leaves room for the result
    import torch

    from paper_2510_09813_b200 import workloads

    reg, seq = workloads.config("random29")
    s = rs.HamiltonianSlice.from_parameters(*seq.step(40), rs.interaction_matrix(reg))
    psi = torch.zeros(2 ** 29, dtype=torch.complex128, device="cuda")
    psi[0] = 1.0
    out, rep = rs.expm_multiply(s, psi, 10.0, rs.KrylovConfig(1e-10))
    assert rep.converged and tuple(out.shape) == (2 ** 29,)
    assert abs(math.sqrt(rs.overlap(out, out).real) - 1.0) <= 1e-9
    del out, psi
    torch.cuda.empty_cache()


class TestDense:
    """hamiltonian.py:191 build_dense (the reference's small-N oracle helper): Hermitian, equal to the
    structured apply column by column, refused above the cap."""

    def test_dense_matches_structured_apply(self, rs):
        rng = np.random.default_rng(191)
        n = 8
        reg = chain(rs, n, 6.0)
        u = rs.interaction_matrix(reg)
        om, de = rng.uniform(0.5, 3.0, n), rng.uniform(-2.0, 2.0, n)
        sl = rs.HamiltonianSlice.from_parameters(om, de, u)
        h = rs.build_dense(sl)
        assert np.array_equal(h, h.conj().T)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
        assert np.linalg.norm(h @ psi - ref) <= 1e-12 * np.linalg.norm(ref)
        assert np.linalg.norm(h @ psi - host(rs.apply_hamiltonian(sl, psi))) <= 1e-12 * np.linalg.norm(ref)

    def test_dense_refused_above_cap(self, rs):
        from paper_2510_09813_b200.hamiltonian import DENSE_QUBIT_CAP

        n = DENSE_QUBIT_CAP + 1
        sl = rs.HamiltonianSlice.from_parameters(np.ones(n), np.zeros(n), np.zeros((n, n)))
        with pytest.raises(rs.ValidationError):
            rs.build_dense(sl)
