"""Pin the CPU oracle (oracle/sv_oracle.py) to the reference's own outputs (tests/golden/*.npz).

CPU-only. The golden vectors were produced by running the real reference
(rydsim, /root/reference/pkg/src) with tests/golden/make_golden.py.
"""

import os

import numpy as np
import pytest

from oracle import sv_oracle as O

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name))


class TestHamiltonianOracle:
    def test_apply_matches_reference(self):
        g = load("apply_hamiltonian.npz")
        for n in (1, 2, 3, 4, 5, 7, 8, 10, 11, 12, 13):
            om, de, u = g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"]
            diag = O.build_diagonal(de, u)
            assert np.abs(diag - g[f"n{n}_diag"]).max() <= 1e-12 * max(1.0, np.abs(diag).max())
            out = O.apply_hamiltonian(om, diag, g[f"n{n}_psi"])
            ref = g[f"n{n}_hpsi"]
            assert np.abs(out - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), n

    def test_diagonal_known_answers(self):
        g = load("diagonal.npz")
        for n in (1, 2, 6, 9):
            d = O.build_diagonal(g[f"n{n}_deltas"], g[f"n{n}_u"])
            assert np.array_equal(d, g[f"n{n}_diag"])
        u = g["line3_u"]
        assert u[0, 1] == pytest.approx(320.0) and u[0, 2] == pytest.approx(5.0)
        # spec examples (SPEC rydberg-hamiltonian build_diagonal)
        assert O.build_diagonal([2.5], np.zeros((1, 1))).tolist() == [0.0, -2.5]
        uu = np.array([[0.0, 7.0], [7.0, 0.0]])
        assert O.build_diagonal([1.0, 2.0], uu).tolist() == [0.0, -1.0, -2.0, 4.0]
        assert O.weighted_bit_sum([1.0, 10.0, 100.0]).tolist() == [0, 1, 10, 11, 100, 101, 110, 111]

    def test_interaction_matrix(self):
        u = O.interaction_matrix([(0.0, 0.0), (3.0, 4.0)], 100.0)
        assert u[0, 1] == pytest.approx(100.0 / 5.0 ** 6)
        with pytest.raises(O.OracleError):
            O.interaction_matrix([(1.0, 2.0), (1.0, 2.0)], 1.0)


class TestKrylovOracle:
    def test_expm_matches_reference(self):
        g = load("expm_multiply.npz")
        for n in range(2, 11):
            om, de, u = g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"]
            diag = O.build_diagonal(de, u)
            out, it, conv, res, _, _ = O.expm_multiply(
                lambda v: O.apply_hamiltonian(om, diag, v), g[f"n{n}_psi"], float(g[f"n{n}_dt"]), 1e-10)
            assert conv and it == int(g[f"n{n}_iterations"])
            assert np.linalg.norm(out - g[f"n{n}_out"]) <= 1e-12

    def test_rabi_and_edge_cases(self):
        h = 0.5 * 2 * np.pi * np.array([[0.0, 1.0], [1.0, 0.0]])
        out, it, conv, *_ = O.expm_multiply(lambda v: h @ v, np.array([1.0, 0.0], complex), 125.0, 1e-12)
        half = 0.5 * 2 * np.pi * 0.125
        assert np.linalg.norm(out - [np.cos(half), -1j * np.sin(half)]) <= 1e-12
        z = np.zeros(4, complex)
        assert O.expm_multiply(lambda v: v, z, 5.0)[1] == 0
        assert O.expm_multiply(lambda v: v, np.array([0.6, 0.8j]), 0.0)[1] == 1

    def test_plain_three_term_recurrence_agrees(self):
        # the fused GPU recurrence does not re-orthogonalise: the oracle shows that
        # the plain three-term Lanczos meets the same tolerance on these inputs
        g = load("expm_multiply.npz")
        for n in (6, 8, 10):
            om, de, u = g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"]
            diag = O.build_diagonal(de, u)
            out, *_ = O.expm_multiply(lambda v: O.apply_hamiltonian(om, diag, v), g[f"n{n}_psi"],
                                      float(g[f"n{n}_dt"]), 1e-10, full_reorth=False)
            assert np.linalg.norm(out - g[f"n{n}_out"]) <= 1e-9


class TestEvolveOracle:
    @pytest.mark.parametrize("case", ["ring10", "adiabatic5", "adiabatic9", "random0", "random1", "random2",
                                      "blockade2", "detmap12"])
    def test_evolve_matches_reference(self, case):
        g = load(f"evolve_{case}.npz")
        u = O.interaction_matrix(g["positions"], float(g["c6"]))
        assert np.abs(u - g["u"]).max() <= 1e-9 * max(1.0, np.abs(u).max())
        res = O.evolve_sv(g["omegas"], g["deltas"], int(g["dt"]), u, tolerance=float(g["tol"]),
                          observe_every=int(g["every"]))
        assert np.linalg.norm(res["final_state"] - g["final_state"]) <= 1e-10
        occ = np.array([r[2] for r in res["occupations"]])
        assert np.abs(occ - g["occ"]).max() <= 1e-10
        assert res["iterations"] == list(g["iterations"])

    def test_dense_oracle_agrees(self):
        g = load("evolve_random0.npz")
        u = g["u"]
        psi = O.evolve_dense(g["omegas"], g["deltas"], int(g["dt"]), u)
        assert np.linalg.norm(psi - g["final_state"]) <= 1e-9


class TestPulsesOracle:
    def test_sampling_and_discretization(self):
        g = load("pulses.npz")
        om, de = O.adiabatic_channels(3, duration_ns=120)
        s_om = O.sample_channels(om, 120)
        s_de = O.sample_channels(de, 120)
        assert np.abs(s_om - g["adiabatic_omega"]).max() <= 1e-12
        assert np.abs(s_de - g["adiabatic_delta"]).max() <= 1e-12
        assert np.abs(O.discretize(s_om, 8) - g["adiabatic_disc_omega_dt8"]).max() <= 1e-12
        assert np.abs(O.discretize(s_de, 8) - g["adiabatic_disc_delta_dt8"]).max() <= 1e-12
        rng = np.random.default_rng(5)
        om, de = O.random_channels(rng, 3, 60)
        s = O.sample_channels(om, 60)
        assert np.abs(s - g["random_omega"]).max() <= 1e-12
        assert np.abs(O.sample_channels(de, 60) - g["random_delta"]).max() <= 1e-12
        assert np.abs(O.discretize(s, 1) - g["random_disc_omega_dt1"]).max() <= 1e-12

    def test_spec_examples(self):
        x = np.arange(8, dtype=float)[None, :]
        assert O.discretize(x, 4)[:, 0].tolist() == [2.0, 6.0]
        x = np.arange(10, dtype=float)[None, :]
        assert O.discretize(x, 5)[:, 0].tolist() == [2.5, 7.5]
        x = np.array([[0.0, 1.0, 2.0, 3.0]])
        assert O.discretize(x, 1)[:, 0].tolist() == [0.5, 1.5, 2.5, 3.0]
        assert O.memory_estimate_sv(1, 1) == 96
        assert O.memory_estimate_sv(26, 15) < 20e9


class TestSamplingOracle:
    def test_sampling_matches_reference(self):
        g = load("sampling.npz")
        for n in (1, 5, 10, 14):
            idx = O.sample_bitstrings(g[f"n{n}_psi"], int(g[f"n{n}_shots"]), int(g[f"n{n}_seed"]))
            assert np.array_equal(idx, g[f"n{n}_idx"]), n

    def test_reference_uniform_streams(self):
        # the host half of the device sampler draws exactly the reference's uniforms
        from paper_2510_09813_b200.observables import sample_uniforms

        g = load("sampling.npz")
        psi = g["n10_psi"]
        cdf = np.cumsum(np.abs(psi) ** 2 / np.sum(np.abs(psi) ** 2))
        cdf[-1] = 1.0
        u = sample_uniforms(int(g["n10_shots"]), int(g["n10_seed"]))
        assert np.array_equal(np.searchsorted(cdf, u, side="right"), g["n10_idx"])


class TestHostLanczosOracle:
    """oracle/big.py (the reference's Lanczos loop on the host with the C matvec and in-place C vector
    operations, used for the N=27/29 GPU parity tests) against the reference's golden vectors and the
    numpy restatement."""

    def test_c_matvec_matches_reference(self):
        from oracle import big

        g = load("apply_hamiltonian.npz")
        for n in (1, 2, 3, 5, 8, 10, 13):
            h = big.HostHamiltonian(g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"])
            assert np.abs(h.diag - g[f"n{n}_diag"]).max() <= 1e-12 * max(1.0, np.abs(h.diag).max())
            psi = np.ascontiguousarray(g[f"n{n}_psi"], dtype=np.complex128)
            out = h.matvec(psi, np.empty_like(psi))
            ref = g[f"n{n}_hpsi"]
            assert np.abs(out - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), n
            part = np.zeros_like(psi)
            lo, hi = len(psi) // 3, len(psi) // 3 + max(1, len(psi) // 4)
            h.matvec_range(psi, part, lo, hi)
            assert np.array_equal(part[lo:hi], out[lo:hi])

    def test_expm_matches_reference_golden(self):
        from oracle import big

        g = load("expm_multiply.npz")
        for n in range(2, 11):
            h = big.HostHamiltonian(g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"])
            out, it, conv, res, _, _ = big.expm_multiply(h, g[f"n{n}_psi"], float(g[f"n{n}_dt"]), 1e-10)
            assert conv and it == int(g[f"n{n}_iterations"]), n
            assert np.linalg.norm(out - g[f"n{n}_out"]) <= 1e-12, n

    def test_expm_matches_numpy_restatement(self):
        from oracle import big

        rng = np.random.default_rng(21)
        n = 12
        om, de = rng.uniform(0, 4, n), rng.uniform(-3, 3, n)
        u = np.triu(rng.uniform(0, 2, (n, n)), 1)
        u = u + u.T
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        h = big.HostHamiltonian(om, de, u)
        a = big.expm_multiply(h, psi, 12.0, 1e-11)
        diag = O.build_diagonal(de, u)
        b = O.expm_multiply(lambda v: O.apply_hamiltonian(om, diag, v), psi, 12.0, 1e-11)
        assert a[1] == b[1] and a[2] and b[2]
        assert np.allclose(a[4], b[4], rtol=1e-12, atol=1e-12) and np.allclose(a[5], b[5], rtol=1e-11)
        assert np.linalg.norm(a[0] - b[0]) <= 1e-12 * np.linalg.norm(psi)
        with pytest.raises(O.OracleError):
            big.expm_multiply(h, psi, 12.0, 1e-11, max_vectors=3)
        z = big.expm_multiply(h, np.zeros(2 ** n, complex), 12.0)
        assert z[1] == 0 and z[2]
