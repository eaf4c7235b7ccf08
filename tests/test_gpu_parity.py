"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and the
CPU oracle on the same seeded inputs. Tolerances are written per test:

* H.psi: relative 1e-12 of max |H psi| (reference: hamiltonian tests use 1e-12);
* Lanczos step: ||out - ref|| <= 100 p (krylov.py tests), p = Krylov tolerance;
* evolution: fidelity 1 - |<ref|gpu>|^2 <= 1e-10 and observables within 1e-8 absolute
  (north-star acceptance), plus ||out - ref|| <= 1e-8.
"""

import math
import os

import numpy as np
import pytest

from oracle import sv_oracle as O

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def load(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="module")
def rs():
    import paper_2510_09813_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


def random_slice(rng, n):
    om = rng.uniform(0.0, 4.0, n)
    de = rng.uniform(-3.0, 3.0, n)
    u = np.triu(rng.uniform(0.0, 2.0, (n, n)), 1)
    return om, de, u + u.T


def rel_err(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


class TestApplyHamiltonian:
    def test_golden_vectors(self, rs):
        g = load("apply_hamiltonian.npz")
        for n in (1, 2, 3, 4, 5, 7, 8, 10, 11, 12, 13):
            s = rs.HamiltonianSlice.from_parameters(g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"])
            out = rs.apply_hamiltonian(s, g[f"n{n}_psi"])
            assert rel_err(out, g[f"n{n}_hpsi"]) <= 1e-12, n

    def test_explicit_diagonal_vec_mode(self, rs):
        g = load("apply_hamiltonian.npz")
        for n in (3, 10, 13):
            s = rs.HamiltonianSlice(g[f"n{n}_omegas"], g[f"n{n}_diag"])
            out = rs.apply_hamiltonian(s, g[f"n{n}_psi"])
            assert rel_err(out, g[f"n{n}_hpsi"]) <= 1e-12, n

    @pytest.mark.parametrize("n", [14, 20, 23])
    def test_explicit_diagonal_vec_mode_multi_pass(self, rs, torch, n):
        # diag="vec" with a multi-pass plan: the lo pass (4096-amplitude contiguous tiles) stages the
        # diagonal tile in shared memory by a bulk copy (RSV_DVEC_SMEM); against the oracle
        rng = np.random.default_rng(500 + n)
        om, de, u = random_slice(rng, n)
        diag = O.build_diagonal(de, u)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        ref = O.apply_hamiltonian(om, diag, psi)
        s = rs.HamiltonianSlice(om, diag)
        out = rs.apply_hamiltonian(s, torch.from_numpy(psi).cuda()).cpu().numpy()
        assert rel_err(out, ref) <= 1e-12

    @pytest.mark.parametrize("n", [14, 17, 20, 22, 23, 24])
    def test_multi_pass_against_oracle(self, rs, torch, n):
        # 13..22 qubits: lo pass + 1 group pass; >= 23: lo + 2 group passes
        rng = np.random.default_rng(n)
        om, de, u = random_slice(rng, n)
        om[n // 2] = 0.0   # a zero drive is skipped by the kernel
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        out = rs.apply_hamiltonian(s, torch.from_numpy(psi).cuda()).cpu().numpy()
        assert rel_err(out, ref) <= 1e-12

    @pytest.mark.parametrize("n", [21, 25, 26, 27, 28])
    def test_plan_shapes_against_c_matvec(self, rs, torch, n):
        # N=21: one 9-bit group pass (a=3, g=9: the 5-D tensor map's second group dimension);
        # 25..28: lo + two groups of 6..8 bits (every plan shape below the N=29/30 ones, which
        # tests/test_headline_parity_gpu.py covers); checked over the whole vector against the
        # C restatement of the reference's compiled matvec (rydsim/_kernels.py:13)
        from oracle import big

        rng = np.random.default_rng(100 + n)
        om, de, u = random_slice(rng, n)
        om[3] = 0.0
        gen = torch.Generator(device="cuda").manual_seed(n)
        x = torch.randn(2 ** n, dtype=torch.complex128, device="cuda", generator=gen)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        out = rs.apply_hamiltonian(s, x).cpu().numpy()
        psi = x.cpu().numpy()
        del x
        ref = big.HostHamiltonian(om, de, u).matvec(psi, np.empty_like(psi))
        assert rel_err(out, ref) <= 1e-12
        if n == 21:
            assert [(p["a"], p["g"]) for p in rs.hamiltonian.context_for(n, u).pass_plan()] == [(12, 0), (3, 9)]

    def test_build_diagonal_on_device(self, rs):
        g = load("diagonal.npz")
        for n in (1, 2, 6, 9):
            d = rs.build_diagonal(g[f"n{n}_deltas"], g[f"n{n}_u"])
            assert isinstance(d, np.ndarray)   # numpy, like the reference (hamiltonian.py:114)
            assert np.abs(d - g[f"n{n}_diag"]).max() <= 1e-12 * max(1, np.abs(d).max())
            dd = rs.build_diagonal(g[f"n{n}_deltas"], g[f"n{n}_u"], device=True)
            assert dd.is_cuda and np.array_equal(dd.cpu().numpy(), d)

    def test_reference_diagonal_helpers_and_lazy_slice_diagonal(self, rs):
        # hamiltonian.py:83 weighted_bit_sum, :99 interaction_diagonal, :131 slice.diagonal
        assert rs.weighted_bit_sum([1.0, 10.0, 100.0]).tolist() == [0, 1, 10, 11, 100, 101, 110, 111]
        g = load("apply_hamiltonian.npz")
        for n in (3, 10):
            om, de, u = g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"]
            idiag = rs.interaction_diagonal(u)
            assert np.abs(idiag - O.interaction_diagonal(u)).max() <= 1e-12 * max(1.0, np.abs(idiag).max())
            assert np.abs(rs.weighted_bit_sum(-de) + idiag - g[f"n{n}_diag"]).max() <= 1e-12 * max(1.0, np.abs(idiag).max())
            s = rs.HamiltonianSlice.from_parameters(om, de, u)
            assert s.structured and isinstance(s.diagonal, np.ndarray)
            assert np.abs(s.diagonal - g[f"n{n}_diag"]).max() <= 1e-12 * max(1.0, np.abs(idiag).max())
            # force_numpy is accepted (the reference's cross-check flag); same CUDA result
            a = rs.apply_hamiltonian(s, g[f"n{n}_psi"])
            b = rs.apply_hamiltonian(s, g[f"n{n}_psi"], force_numpy=True)
            assert np.array_equal(a, b) and rel_err(a, g[f"n{n}_hpsi"]) <= 1e-12
        with pytest.raises(rs.ValidationError):
            rs.HamiltonianSlice([1.0, 2.0], np.zeros(3))

    def test_linearity_and_hermiticity_large(self, rs, torch):
        n = 26
        rng = np.random.default_rng(3)
        om, de, u = random_slice(rng, n)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        gen = torch.Generator(device="cuda").manual_seed(1)
        x = torch.randn(2 ** n, dtype=torch.complex128, device="cuda", generator=gen)
        y = torch.randn(2 ** n, dtype=torch.complex128, device="cuda", generator=gen)
        hx = rs.apply_hamiltonian(s, x)
        hy = rs.apply_hamiltonian(s, y)
        # <y|Hx> = conj(<x|Hy>) for Hermitian H (size-independent property)
        a = rs.overlap(y, hx)
        b = rs.overlap(x, hy).conjugate()
        assert abs(a - b) <= 1e-10 * abs(a)
        e = rs.overlap(x, hx)
        assert abs(e.imag) <= 1e-10 * abs(e.real)


class TestExpm:
    def test_golden_lanczos_steps(self, rs):
        g = load("expm_multiply.npz")
        p = 1e-10
        for n in range(2, 11):
            s = rs.HamiltonianSlice.from_parameters(g[f"n{n}_omegas"], g[f"n{n}_deltas"], g[f"n{n}_u"])
            out, rep = rs.expm_multiply(s, g[f"n{n}_psi"], float(g[f"n{n}_dt"]), rs.KrylovConfig(p))
            assert rep.converged
            assert np.linalg.norm(out - g[f"n{n}_out"]) <= 100 * p, n
            assert abs(rep.iterations - int(g[f"n{n}_iterations"])) <= 1

    def test_generic_callable_path(self, rs, torch):
        lam = torch.linspace(-5, 5, 64, dtype=torch.float64, device="cuda")
        rng = np.random.default_rng(0)
        psi = torch.from_numpy(rng.standard_normal(64) + 1j * rng.standard_normal(64)).cuda()
        out, rep = rs.expm_multiply(lambda v: lam * v, psi, 150.0, rs.KrylovConfig(1e-12))
        exp = torch.exp(-1j * lam * 0.150) * psi
        assert rep.converged and (out - exp).abs().max().item() <= 1e-11

    def test_edge_cases(self, rs):
        s = rs.HamiltonianSlice.from_parameters([1.0, 2.0], [0.3, -0.2], np.array([[0, 3.0], [3.0, 0]]))
        psi = np.array([0.5, 0.5j, -0.5, 0.5], dtype=complex)
        out, rep = rs.expm_multiply(s, psi, 0.0)
        assert np.array_equal(out, psi) and rep.iterations == 1 and rep.converged
        out, rep = rs.expm_multiply(s, np.zeros(4, complex), 10.0)
        assert rep.iterations == 0 and rep.converged and not np.any(out)
        # eigenvector terminates early: |00> with zero drive
        s0 = rs.HamiltonianSlice.from_parameters([0.0, 0.0], [0.3, -0.2], np.zeros((2, 2)))
        out, rep = rs.expm_multiply(s0, np.array([0, 1, 0, 0], complex), 100.0, rs.KrylovConfig(1e-12))
        assert rep.converged and rep.iterations <= 2
        assert abs(out[1] - np.exp(1j * 0.3 * 0.1)) <= 1e-12

    def test_forward_backward_large(self, rs, torch):
        n = 24
        rng = np.random.default_rng(5)
        om, de, u = random_slice(rng, n)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        gen = torch.Generator(device="cuda").manual_seed(2)
        psi = torch.randn(2 ** n, dtype=torch.complex128, device="cuda", generator=gen)
        psi /= torch.linalg.vector_norm(psi)
        fwd, r1 = rs.expm_multiply(s, psi, 5.0, rs.KrylovConfig(1e-12))
        back, r2 = rs.expm_multiply(s, fwd, -5.0, rs.KrylovConfig(1e-12))
        assert r1.converged and r2.converged
        assert abs(rs.norm_difference(fwd, fwd) ) == 0.0
        assert rs.norm_difference(back, psi) <= 1e-9
        assert abs(math.sqrt(abs(rs.overlap(fwd, fwd))) - 1.0) <= 1e-10


def run_gpu(rs, g, every, pairs=(), energy=False, diag="fly"):
    n = g["omegas"].shape[1]
    reg = rs.Register(tuple(map(tuple, g["positions"])), float(g["c6"]))
    seq = rs.DiscretizedSequence(int(g["dt"]), g["omegas"], g["deltas"], int(g["dt"]) * g["omegas"].shape[0])
    specs = [rs.ObservableSpec("occupation", (), every)]
    if len(pairs):
        specs.append(rs.ObservableSpec("correlation", tuple(int(q) for p in pairs for q in p), 0))
    if energy:
        specs.append(rs.ObservableSpec("energy", (), 0))
    cfg = rs.SvRunConfig(krylov=rs.KrylovConfig(float(g["tol"])), observables=tuple(specs), diag=diag)
    return rs.evolve_sv(seq, reg, cfg)


class TestEvolve:
    @pytest.mark.parametrize("case", ["ring10", "adiabatic5", "adiabatic9", "random0", "random1", "random2",
                                      "blockade2", "detmap12"])
    @pytest.mark.parametrize("diag", ["fly", "vec"])
    def test_golden_evolutions(self, rs, case, diag):
        g = load(f"evolve_{case}.npz")
        pairs = g["pairs"] if "pairs" in g.files else ()
        res = run_gpu(rs, g, int(g["every"]), pairs, energy=True, diag=diag)
        psi = res.final_state.cpu().numpy()
        ref = g["final_state"]
        fid = abs(np.vdot(ref, psi)) ** 2
        assert 1.0 - fid <= 1e-10
        assert np.linalg.norm(psi - ref) <= 1e-8
        occ = np.array([r.values for r in res.observables if r.kind == "occupation"])
        assert occ.shape == g["occ"].shape
        assert np.abs(occ - g["occ"]).max() <= 1e-8
        if len(pairs):
            corr = [r.values for r in res.observables if r.kind == "correlation"][-1]
            assert np.abs(np.array(corr) - g["corr"]).max() <= 1e-8
        e = [r.values[0] for r in res.observables if r.kind == "energy"][-1]
        assert abs(e - float(g["energy_last"])) <= 1e-8 * max(1.0, abs(float(g["energy_last"])))
        iters = np.array([r.iterations for r in res.krylov_reports])
        assert np.abs(iters - g["iterations"]).max() <= 1

    def test_lattice20_config1(self, rs):
        g = load("evolve_lattice20.npz")
        res = run_gpu(rs, g, 1)
        psi = res.final_state.cpu().numpy()
        rng = np.random.default_rng(77)
        probe = rng.standard_normal(2 ** 20) + 1j * rng.standard_normal(2 ** 20)
        assert abs(np.vdot(probe, psi) - complex(g["probe_overlap"])) <= 1e-8 * abs(complex(g["probe_overlap"]))
        assert np.abs(psi[:64] - g["amp_head"]).max() <= 1e-9
        occ = np.array([r.values for r in res.observables])
        assert np.abs(occ - g["occ"]).max() <= 1e-8

    def test_lattice20_config1_full_sweep(self, rs):
        # BASELINE configs[1] for its whole length: the 3 us adiabatic sweep (300 steps of 10 ns)
        # against the reference's own run (tests/golden/make_golden.py --lattice20-full)
        g = load("evolve_lattice20_full.npz")
        res = run_gpu(rs, g, int(g["every"]), energy=True)
        psi = res.final_state.cpu().numpy()
        rng = np.random.default_rng(77)
        probe = rng.standard_normal(2 ** 20) + 1j * rng.standard_normal(2 ** 20)
        assert abs(np.vdot(probe, psi) - complex(g["probe_overlap"])) <= 1e-8 * abs(complex(g["probe_overlap"]))
        assert np.abs(psi[:64] - g["amp_head"]).max() <= 1e-9
        assert np.abs(psi[-64:] - g["amp_tail"]).max() <= 1e-9
        occ = np.array([r.values for r in res.observables if r.kind == "occupation"])
        assert occ.shape == g["occ"].shape
        assert np.abs(occ - g["occ"]).max() <= 1e-8
        e = [r.values[0] for r in res.observables if r.kind == "energy"][-1]
        assert abs(e - float(g["energy_last"])) <= 1e-8 * max(1.0, abs(float(g["energy_last"])))
        iters = np.array([r.iterations for r in res.krylov_reports])
        assert len(iters) == 300 and np.abs(iters - g["iterations"]).max() <= 1

    def test_krylov_cap_substepping_is_exact(self, rs, torch):
        # a tiny HBM budget caps the resident Krylov basis; the step is split in time (tail
        # regeneration off) and must agree
        from paper_2510_09813_b200.engine import SvEngine

        g = load("evolve_detmap12.npz")
        n = 12
        reg = rs.Register(tuple(map(tuple, g["positions"])), float(g["c6"]))
        u = rs.interaction_matrix(reg)
        full = SvEngine(n, u, krylov_vectors_cap=60)
        capped = SvEngine(n, u, krylov_vectors_cap=6)
        capped.set_tail_regeneration(False)
        subs = 0
        for k in range(5):
            full.step(g["omegas"][k], g["deltas"][k], 10.0, 1e-12, 100)
            subs += capped.step(g["omegas"][k], g["deltas"][k], 10.0, 1e-12, 100).substeps
        assert subs > 0
        assert rs.norm_difference(full.state(), capped.state()) <= 1e-9

    @pytest.mark.parametrize("n,cap", [(12, 4), (12, 6), (22, 4), (22, 7)])
    def test_tail_regeneration_matches_resident_basis(self, rs, torch, n, cap):
        # beyond the resident basis the recurrence continues in a two-slot ring and the overwritten
        # vectors are regenerated for the combination: same Krylov dimension per step as with the
        # whole basis resident (the reference's k, krylov.py:96-117) and the same state to rounding
        from paper_2510_09813_b200.engine import SvEngine

        rng = np.random.default_rng(n + cap)
        om, de, u = random_slice(rng, n)
        full = SvEngine(n, u, krylov_vectors_cap=60)
        capped = SvEngine(n, u, krylov_vectors_cap=cap)
        for e in (full, capped):
            e.set_speculation(0)
        full.set_observables([1 << q for q in range(n)])
        capped.set_observables([1 << q for q in range(n)])
        regen = 0
        for k in range(4):
            dt = 6.0 + 3.0 * k
            a = full.step(om, de, dt, 1e-12, 100, next_params=(om, de), observe=True)
            b = capped.step(om, de, dt, 1e-12, 100, next_params=(om, de), observe=True)
            assert a.converged and b.converged and b.substeps == 0
            assert a.iterations == b.iterations and a.iterations > cap
            assert b.regenerated == a.iterations - cap and b.matvecs == a.matvecs + b.regenerated
            assert abs(a.alpha0 - b.alpha0) <= 1e-12 * max(1.0, abs(a.alpha0))
            assert np.abs(full.observables() - capped.observables()).max() <= 1e-13
            regen += b.regenerated
        assert regen > 0
        assert rs.norm_difference(full.state(), capped.state()) <= 1e-12
        for e in (full, capped):
            e.close()

    @pytest.mark.parametrize("n", [22, 24])
    def test_vec_diagonal_matches_fly(self, rs, torch, n):
        # Lanczos steps with the precomputed interaction diagonal (lo pass reads it from shared memory,
        # staged per tile) against the on-the-fly diagonal: same Krylov dimensions, same state to rounding
        from paper_2510_09813_b200.engine import SvEngine

        rng = np.random.default_rng(70 + n)
        om, de, u = random_slice(rng, n)
        engines = [SvEngine(n, u, diag=d, krylov_vectors_cap=40) for d in ("fly", "vec")]
        psi0 = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        psi0 /= np.linalg.norm(psi0)
        for e in engines:
            e.set_state(torch.from_numpy(psi0).cuda())
            e.set_observables([1 << q for q in range(n)])
        for k in range(3):
            a, b = (e.step(om, de, 4.0 + k, 1e-10, 100, next_params=(om, de), observe=True) for e in engines)
            assert a.iterations == b.iterations
            assert abs(a.alpha0 - b.alpha0) <= 1e-11 * max(1.0, abs(a.alpha0))
            assert np.abs(engines[0].observables() - engines[1].observables()).max() <= 1e-12
        assert rs.norm_difference(engines[0].state(), engines[1].state()) <= 1e-11
        for e in engines:
            e.close()

    @pytest.mark.parametrize("n", [10, 20])
    def test_speculative_iterations_change_nothing(self, rs, torch, n):
        # iteration j+1 launched before the host tests j (small N): the same kernels in the same
        # order, so the same state bit for bit; the discarded iteration is not counted
        from paper_2510_09813_b200.engine import SvEngine

        rng = np.random.default_rng(40 + n)
        om, de, u = random_slice(rng, n)
        runs = []
        for mode in (0, 1):
            e = SvEngine(n, u, krylov_vectors_cap=60)
            e.set_speculation(mode)
            reps = [e.step(om, de, 5.0 + k, 1e-10, 100, next_params=(om, de)) for k in range(5)]
            runs.append((e.state().cpu().numpy(), [(r.iterations, r.matvecs) for r in reps]))
            e.close()
        assert np.array_equal(runs[0][0], runs[1][0])
        assert runs[0][1] == runs[1][1]

    def test_sampled_kernel_timing(self, rs, torch):
        # rsv_set_profiling(ctx, P) times one launch in P per kernel family: every launch is counted,
        # the reported time is the timed launches' mean times the count, and the state is unchanged
        from paper_2510_09813_b200.engine import SvEngine

        rng = np.random.default_rng(77)
        om, de, u = random_slice(rng, 18)
        out = {}
        for every in (1, 4):
            e = SvEngine(18, u, krylov_vectors_cap=60)
            e.set_profiling(True, every=every)
            reps = [e.step(om, de, 5.0 + k, 1e-10, 100, next_params=(om, de)) for k in range(4)]
            prof = e.profile()
            out[every] = (e.state().cpu().numpy(), prof, sum(r.matvecs for r in reps))
            e.close()
        assert np.array_equal(out[1][0], out[4][0])
        for every in (1, 4):
            prof, mv = out[every][1], out[every][2]
            first = next(iter(prof))
            assert prof[first]["launches"] >= mv and prof[first]["ms"] > 0.0
            assert prof["combine"]["launches"] >= 4   # + the first step's q_0 preparation
        for fam in out[1][1]:
            assert out[1][1][fam]["launches"] == out[4][1][fam]["launches"]

    @pytest.mark.parametrize("n", [16, 18, 21])
    def test_fused_iteration_matches_separate_passes(self, rs, torch, n):
        # [lo, last] plans with 4096-amplitude tiles (16..21 qubits) run each Lanczos iteration as one cooperative launch
        # (iter2_kernel: lo pass, grid barrier, last pass); against the two separate launches
        from paper_2510_09813_b200.engine import SvEngine

        rng = np.random.default_rng(60 + n)
        om, de, u = random_slice(rng, n)
        runs = []
        for mode in (0, 1):
            e = SvEngine(n, u, krylov_vectors_cap=60)
            e.set_fusion(mode)
            assert e.pass_plan()[0]["family"] == ("iter2" if mode else "lo")
            e.set_observables([1 << q for q in range(n)])
            reps = [e.step(om, de, 5.0 + k, 1e-10, 100, next_params=(om, de), observe=True) for k in range(4)]
            runs.append((e.state().cpu().numpy(), [(r.iterations, r.matvecs) for r in reps], e.observables(),
                         reps[-1].alpha0))
            e.close()
        assert runs[0][1] == runs[1][1]
        assert np.linalg.norm(runs[0][0] - runs[1][0]) <= 1e-11
        assert np.abs(runs[0][2] - runs[1][2]).max() <= 1e-12
        assert abs(runs[0][3] - runs[1][3]) <= 1e-11 * max(1.0, abs(runs[0][3]))

    def test_host_final_state_and_force_numpy_flag(self, rs):
        # SvRunConfig(host_final_state=True): numpy final state like the reference (sv.py:66), the
        # workspace released; force_numpy_matvec (sv.py:61) is accepted and changes nothing
        g = load("evolve_ring10.npz")
        reg = rs.Register(tuple(map(tuple, g["positions"])), float(g["c6"]))
        seq = rs.DiscretizedSequence(int(g["dt"]), g["omegas"][:8], g["deltas"][:8], 8 * int(g["dt"]))
        a = rs.evolve_sv(seq, reg, rs.SvRunConfig(krylov=rs.KrylovConfig(1e-10)))
        b = rs.evolve_sv(seq, reg, rs.SvRunConfig(krylov=rs.KrylovConfig(1e-10), host_final_state=True,
                                                  force_numpy_matvec=True))
        assert isinstance(b.final_state, np.ndarray) and b.engine is None
        assert np.array_equal(a.final_state.cpu().numpy(), b.final_state)

    def test_rabi_analytic(self, rs):
        seq = rs.discretize(rs.sample_program(rs.ChannelProgram.from_channels(
            [[rs.Constant(500, 2 * np.pi)]], [[rs.Constant(500, 0.0)]], 500)), 1)
        reg = rs.Register(((0.0, 0.0),), 1.0)
        res = rs.evolve_sv(seq, reg, rs.SvRunConfig(krylov=rs.KrylovConfig(1e-12),
                                                    observables=(rs.ObservableSpec("occupation", (0,)),)))
        t = np.array([r.t_ns for r in res.observables]) * 1e-3
        v = np.array([r.values[0] for r in res.observables])
        assert np.abs(v - np.sin(np.pi * t) ** 2).max() <= 1e-10

    def test_errors(self, rs):
        seq = rs.DiscretizedSequence(10, np.ones((1, 4)), np.zeros((1, 4)), 10)
        reg = rs.Register(tuple((1e6 * i, 0.0) for i in range(4)), 1.0)
        with pytest.raises(rs.ValidationError):
            rs.evolve_sv(seq, reg, rs.SvRunConfig(qubit_cap=3))
        seq2 = rs.DiscretizedSequence(100, np.full((1, 2), 300.0), np.full((1, 2), -500.0), 100)
        reg2 = rs.Register(((0.0, 0.0), (1e6, 0.0)), 1.0)
        with pytest.raises(rs.SolverError) as err:
            rs.evolve_sv(seq2, reg2, rs.SvRunConfig(krylov=rs.KrylovConfig(1e-12, max_krylov_dim=2)))
        assert err.value.step == 0


class TestObservables:
    def test_against_oracle(self, rs):
        rng = np.random.default_rng(4)
        for n in (3, 9, 15):
            psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
            occ = rs.occupations(psi)
            assert np.abs(occ - O.occupations(psi)).max() <= 1e-13
            assert abs(rs.correlation(psi, 0, n - 1) - O.correlation(psi, 0, n - 1)) <= 1e-13
            phi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
            assert abs(rs.overlap(psi, phi) - np.vdot(psi, phi)) <= 1e-10 * abs(np.vdot(psi, phi))
            assert abs(rs.norm_difference(psi, phi) - np.linalg.norm(psi - phi)) <= 1e-12 * np.linalg.norm(psi)


class TestFullSize:
    """BASELINE configs[3] size (N=29) through size-independent properties."""

    @pytest.fixture(scope="class")
    @staticmethod
    def setup29(rs, torch):
        from paper_2510_09813_b200 import workloads
        from paper_2510_09813_b200.engine import SvEngine

        reg, seq = workloads.config("random29")
        u = rs.interaction_matrix(reg)
        eng = SvEngine(29, u, diag="fly", max_krylov_dim=100, krylov_vectors_cap=10)
        yield rs, torch, reg, seq, u, eng
        eng.close()
        del eng
        torch.cuda.empty_cache()

    def test_norm_energy_and_reversibility(self, setup29):
        rs, torch, reg, seq, u, eng = setup29
        for k in range(12):   # into the pulse: a spread-out state
            eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1))
        k = 12
        om, de = seq.step(k)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        psi0 = eng.state().clone()
        h0 = rs.apply_hamiltonian(s, psi0)
        e0 = rs.overlap(psi0, h0).real
        del h0
        rep = eng.step(om, de, 10.0, 1e-10, 100)
        assert rep.converged
        psi1 = eng.state()
        assert abs(math.sqrt(rs.overlap(psi1, psi1).real) - 1.0) <= 1e-9
        h1 = rs.apply_hamiltonian(s, psi1)
        e1 = rs.overlap(psi1, h1).real
        del h1
        assert abs(e1 - e0) <= 1e-8 * max(1.0, abs(e0))
        assert abs(rep.alpha0 - e0) <= 1e-9 * max(1.0, abs(e0))   # Energy observable = alpha_0
        back = eng.step(om, de, -10.0, 1e-10, 100)
        assert back.converged
        assert rs.norm_difference(eng.state(), psi0) <= 1e-8


class TestSampling:
    """Device inverse-CDF sampling (observables.py:167) against the reference's own draws."""

    def test_golden_indices(self, rs, torch):
        g = load("sampling.npz")
        for n in (1, 5, 10, 14):
            psi = torch.from_numpy(g[f"n{n}_psi"]).cuda()
            idx = rs.sample_bitstrings(psi, int(g[f"n{n}_shots"]), int(g[f"n{n}_seed"]))
            assert np.array_equal(idx, g[f"n{n}_idx"]), n

    def test_against_oracle_and_edges(self, rs, torch):
        rng = np.random.default_rng(12)
        for n in (12, 13, 17):   # one chunk, two chunks, many chunks
            psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
            psi[: 2 ** n // 3] = 0.0    # leading zero-probability run
            psi /= np.linalg.norm(psi)
            idx = rs.sample_bitstrings(torch.from_numpy(psi).cuda(), 20000, 99)
            assert np.array_equal(idx, O.sample_bitstrings(psi, 20000, 99)), n
            assert idx.min() >= 2 ** n // 3
        basis = np.zeros(2 ** 15, complex)
        basis[2 ** 15 - 1] = 1.0        # all weight on the last index
        assert np.all(rs.sample_bitstrings(basis, 100, 1) == 2 ** 15 - 1)
        with pytest.raises(rs.ValidationError):
            rs.sample_bitstrings(2 * basis, 10, 1)
        assert np.all(rs.sample_bitstrings(2 * basis, 10, 1, renormalize=True) == 2 ** 15 - 1)
        with pytest.raises(rs.ValidationError):
            rs.sample_bitstrings(basis, 0, 1)

    def test_full_size_histogram(self, rs, torch):
        # N=27 (2^27 amplitudes, 2 GB): per-qubit frequencies of 2^16 shots match the occupations
        n = 27
        gen = torch.Generator(device="cuda").manual_seed(5)
        psi = torch.randn(2 ** n, dtype=torch.complex128, device="cuda", generator=gen)
        psi *= torch.exp(-torch.arange(2 ** n, device="cuda", dtype=torch.float64) / 2 ** 25)
        psi /= torch.linalg.vector_norm(psi)
        shots = 1 << 16
        idx = rs.sample_bitstrings(psi, shots, 17)
        occ = rs.occupations(psi)
        freq = np.array([((idx >> q) & 1).mean() for q in range(n)])
        sigma = np.sqrt(occ * (1 - occ) / shots) + 1e-12
        assert np.all(np.abs(freq - occ) <= 6 * sigma)


class TestReorthogonalization:
    """KrylovConfig(reorthogonalize=True): the fused step re-orthogonalises every Lanczos vector like
    the reference (krylov.py:103-104) -- same acceptance bar, iteration counts as the reference's."""

    @pytest.mark.parametrize("case", ["random1", "detmap12", "adiabatic9"])
    def test_golden_evolutions(self, rs, case):
        g = load(f"evolve_{case}.npz")
        n = g["omegas"].shape[1]
        reg = rs.Register(tuple(map(tuple, g["positions"])), float(g["c6"]))
        seq = rs.DiscretizedSequence(int(g["dt"]), g["omegas"], g["deltas"], int(g["dt"]) * g["omegas"].shape[0])
        cfg = rs.SvRunConfig(krylov=rs.KrylovConfig(float(g["tol"]), reorthogonalize=True),
                             observables=(rs.ObservableSpec("occupation", (), int(g["every"])),))
        res = rs.evolve_sv(seq, reg, cfg)
        psi = res.final_state.cpu().numpy()
        assert 1.0 - abs(np.vdot(g["final_state"], psi)) ** 2 <= 1e-10
        occ = np.array([r.values for r in res.observables])
        assert np.abs(occ - g["occ"]).max() <= 1e-8
        iters = np.array([r.iterations for r in res.krylov_reports])
        assert np.abs(iters - g["iterations"]).max() <= 1

    @pytest.mark.parametrize("n", [14, 22])
    def test_matches_plain_recurrence(self, rs, torch, n):
        rng = np.random.default_rng(n)
        om, de, u = random_slice(rng, n)
        s = rs.HamiltonianSlice.from_parameters(om, de, u)
        psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
        psi /= np.linalg.norm(psi)
        a, ra = rs.expm_multiply(s, psi, 8.0, rs.KrylovConfig(1e-12))
        b, rb = rs.expm_multiply(s, psi, 8.0, rs.KrylovConfig(1e-12, reorthogonalize=True))
        assert ra.converged and rb.converged
        assert np.linalg.norm(a - b) <= 1e-10
        ref = O.expm_multiply(lambda v: O.apply_hamiltonian(om, O.build_diagonal(de, u), v), psi, 8.0, 1e-12)[0]
        assert np.linalg.norm(b - ref) <= 1e-10


class TestMaxSize:
    """N=30, the largest register one B200 holds with a useful Krylov basis (17 GB per vector;
    plan lo + two 9-bit groups with 128 B runs), through size-independent properties."""

    def test_n30_norm_energy_reversibility(self, rs, torch):
        from paper_2510_09813_b200 import workloads
        from paper_2510_09813_b200.engine import SvEngine

        n = 30
        reg, seq = workloads.config("random29", n_override=n)
        u = rs.interaction_matrix(reg)
        eng = SvEngine(n, u, diag="fly", max_krylov_dim=100, krylov_vectors_cap=6)
        try:
            plan = eng.pass_plan()
            assert [p["g"] for p in plan] == [0, 9, 9]
            for k in range(6):
                rep = eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1))
                assert rep.converged
            om, de = seq.step(6)
            psi0 = eng.state().clone()
            rep = eng.step(om, de, 10.0, 1e-10, 100)
            assert rep.converged and rep.regenerated >= 1       # 6 resident vectors: ring + regeneration
            assert abs(math.sqrt(rs.overlap(eng.state(), eng.state()).real) - 1.0) <= 1e-9
            back = eng.step(om, de, -10.0, 1e-10, 100)
            assert back.converged
            assert rs.norm_difference(eng.state(), psi0) <= 1e-8
            assert abs(back.alpha0 - rep.alpha0) <= 1e-9 * max(1.0, abs(rep.alpha0))   # energy conserved
        finally:
            eng.close()
            del eng
            torch.cuda.empty_cache()


class TestFullSizeAlgorithm:
    """N=29: the fused three-term recurrence against the reference's algorithm (full
    re-orthogonalisation) on mid-pulse steps, fidelity 1e-10 and occupations 1e-8 (north star).
    The whole-pulse comparison is tools/full_pulse_parity.py (profiles/r1_full_pulse_parity_n29.json)."""

    def test_three_term_matches_reorthogonalized(self, rs, torch):
        from paper_2510_09813_b200 import workloads
        from paper_2510_09813_b200.engine import SvEngine

        reg, seq = workloads.config("random29")
        u = rs.interaction_matrix(reg)
        host = torch.empty(2 ** 29, dtype=torch.complex128, pin_memory=True)
        occ = []
        for reorth in (False, True):
            eng = SvEngine(29, u, diag="fly", max_krylov_dim=100, krylov_vectors_cap=14)
            eng.set_reorthogonalize(reorth)
            eng.set_observables([1 << q for q in range(29)])
            for k in range(40, 43):
                rep = eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1), observe=True)
                assert rep.converged
            occ.append(eng.observables())
            if not reorth:
                host.copy_(eng.state())
            else:
                other = eng.slots[1]
                other.copy_(host)
                fid = abs(rs.overlap(other, eng.state())) ** 2
            eng.close()
            del eng
            torch.cuda.empty_cache()
        assert 1.0 - fid <= 1e-10
        assert np.abs(occ[0] - occ[1]).max() <= 1e-8
