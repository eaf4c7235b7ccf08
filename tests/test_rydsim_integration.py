"""INTEGRATION.md's switch driven with the REAL reference (rydsim from /root/reference, build container
only) and the device engine mocked by the CPU oracle, so the argument adaptation, result types and
error mapping are checked without a GPU:

* rydsim's own ``execute_run`` (runner.py:179, backend "sv") and ``evolve_sv`` reach this package
  through ``rydsim_plugin.install()`` with RYDSIM_DEVICE=b200, and return rydsim's SvRunResult /
  run document, equal to rydsim's CPU result (the mock runs the reference algorithm);
* a non-converged step raises this package's SolverError, which rydsim's handlers catch as their
  own (rydsim/cli.py:248-258 -> exit code 3); a memory refusal maps to exit code 4.

Each case runs in a subprocess (import order: rydsim first, then this package, as an installed
reference would). Skipped where /root/reference is absent (the GPU box).
"""

import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")

PRELUDE = textwrap.dedent(f"""
    import os, sys, json
    sys.path.insert(0, {REF_SRC!r}); sys.path.insert(0, {ROOT!r})
    import numpy as np
    import rydsim, rydsim.sv, rydsim.runner, rydsim.cli, rydsim.errors
    import paper_2510_09813_b200 as b200
    from paper_2510_09813_b200 import rydsim_plugin, sv as b200_sv
    from oracle import sv_oracle as O

    class FakeTensor:
        def __init__(self, a): self.a = a
        def cpu(self): return self
        def numpy(self): return self.a

    class Rep:
        pass

    class FakeEngine:
        # the SvEngine surface evolve_sv uses, computed by the CPU oracle (reference algorithm)
        fail_at = None
        def __init__(self, n, u, diag="fly", max_krylov_dim=100, device=None, memory_budget_bytes=None,
                     krylov_vectors_cap=None):
            self.n, self.u = n, np.asarray(u)
            self.psi = np.zeros(2 ** n, complex); self.psi[0] = 1.0
            self.masks = []; self.slots = [None]; self.calls = 0
        def set_reorthogonalize(self, on): pass
        def set_state(self, psi): self.psi = np.array(psi, dtype=complex)
        def set_observables(self, masks): self.masks = [int(m) for m in masks]
        def step(self, om, de, dt, tol, kmax, eps=1e-14, next_params=None, observe=False):
            diag = O.build_diagonal(de, self.u)
            out, it, conv, res, alphas, _ = O.expm_multiply(lambda v: O.apply_hamiltonian(om, diag, v),
                                                             self.psi, dt, tol, kmax, eps)
            r = Rep()
            r.iterations, r.residual, r.substeps, r.matvecs, r.regenerated = it, res, 0, it, 0
            r.converged = int(conv and self.calls != FakeEngine.fail_at)
            r.alpha0 = alphas[0] if alphas else 0.0
            r.norm_in = float(np.linalg.norm(self.psi))
            self.calls += 1
            self.psi = out
            return r
        def observables(self):
            p = np.abs(self.psi) ** 2
            idx = np.arange(len(p), dtype=np.uint64)
            return np.array([p[(idx & np.uint64(m)) == np.uint64(m)].sum() / p.sum() for m in self.masks])
        def state(self): return FakeTensor(self.psi)
        def close(self): pass

    b200_sv.SvEngine = FakeEngine
    rydsim_plugin.install()
""")


def run(body):
    code = PRELUDE + textwrap.dedent(body)
    env = dict(os.environ, RYDSIM_DEVICE="b200")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    return p.stdout


def test_errors_derive_from_reference_classes():
    out = run("""
        E = rydsim.errors
        assert b200.REFERENCE_ERRORS
        for name in ("RydsimError", "ValidationError", "ConfigurationError", "SolverError", "MemoryBudgetError"):
            assert issubclass(getattr(b200, name), getattr(E, name)), name
        try:
            raise b200.SolverError("x", step=4, residual=2.0)
        except E.SolverError as err:
            assert err.step == 4 and err.residual == 2.0
        print("ok")
    """)
    assert "ok" in out


def test_evolve_sv_switch_matches_reference_cpu_path():
    out = run("""
        from rydsim.generator import adiabatic_program
        from rydsim.krylov import KrylovConfig
        from rydsim.observables import ObservableSpec
        from rydsim.pulses import discretize, sample_program
        reg, prog = adiabatic_program(5, duration_ns=200)
        seq = discretize(sample_program(prog), 10)
        cfg = rydsim.sv.SvRunConfig(krylov=KrylovConfig(1e-10), snapshot_every=10,
                                    observables=(ObservableSpec("occupation", (), 5),
                                                 ObservableSpec("correlation", (0, 1, 2, 4), 0)))
        ref = rydsim.sv.evolve_sv.__wrapped__(seq, reg, cfg)
        got = rydsim.sv.evolve_sv(seq, reg, cfg)             # RYDSIM_DEVICE=b200: the B200 path
        assert type(got) is rydsim.sv.SvRunResult
        assert isinstance(got.final_state, np.ndarray) and got.final_state.shape == (32,)
        assert np.linalg.norm(got.final_state - ref.final_state) <= 1e-10
        assert [type(r) for r in got.observables] == [rydsim.observables.ObservableRecord] * len(ref.observables)
        for a, b in zip(got.observables, ref.observables):
            assert (a.spec_index, a.kind, a.qubits, a.step, a.t_ns) == (b.spec_index, b.kind, b.qubits, b.step, b.t_ns)
            assert np.abs(np.array(a.values) - np.array(b.values)).max() <= 1e-10
        assert all(type(r) is rydsim.krylov.KrylovReport for r in got.krylov_reports)
        assert [r.iterations for r in got.krylov_reports] == [r.iterations for r in ref.krylov_reports]
        assert [t for t, _ in got.snapshots] == [t for t, _ in ref.snapshots]
        assert got.peak_memory_bytes == ref.peak_memory_bytes and got.dt_ns == ref.dt_ns
        # validation errors keep the reference's class and message
        try:
            rydsim.sv.evolve_sv(seq, reg, rydsim.sv.SvRunConfig(qubit_cap=3))
            raise SystemExit("no error")
        except rydsim.errors.ValidationError as err:
            assert "qubit cap" in str(err)
        print("ok")
    """)
    assert "ok" in out


def test_execute_run_document_through_switch():
    out = run("""
        from rydsim.sequence_io import parse_config, parse_sequence
        cfgs = "/root/reference/pkg/configs"
        reg, prog = parse_sequence(os.path.join(cfgs, "sequence_adiabatic_5q.json"))
        cfg = parse_config(os.path.join(cfgs, "run_sv.json"))
        got = rydsim.runner.execute_run(reg, prog, cfg)      # backend "sv" -> the B200 path
        rydsim_plugin.uninstall()
        ref = rydsim.runner.execute_run(reg, prog, cfg)
        assert got.metadata["backend"] == "sv"
        assert np.linalg.norm(got.final_state - ref.final_state) <= 1e-10
        assert got.data["samples"] == ref.data["samples"]   # same state, same PCG64 draws
        print("ok")
    """)
    assert "ok" in out


def test_cli_exit_codes_for_b200_errors(tmp_path):
    out = run(f"""
        cfgs = "/root/reference/pkg/configs"
        seq = os.path.join(cfgs, "sequence_adiabatic_5q.json")
        FakeEngine.fail_at = 2                                # third step reports non-convergence
        rc = rydsim.cli.main(["run", seq, os.path.join(cfgs, "run_sv.json"), "--out", {str(tmp_path / 'r.json')!r}])
        assert rc == rydsim.cli.EXIT_SOLVER, rc
        FakeEngine.fail_at = None
        def refuse(*a, **k):
            raise b200.MemoryBudgetError("no room", required_bytes=1, budget_bytes=0)
        b200_sv.SvEngine = refuse
        rc = rydsim.cli.main(["run", seq, os.path.join(cfgs, "run_sv.json"), "--out", {str(tmp_path / 'r.json')!r}])
        assert rc == rydsim.cli.EXIT_MEMORY, rc
        print("ok")
    """)
    assert "ok" in out
