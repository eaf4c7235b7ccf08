"""execute_run (runner.py:179, backend "sv") on the B200 path against documents produced by the
reference's own execute_run on its configs/ fixtures (tests/golden/runs_sv.json, make_golden.py
--runs). Tolerances: observables 1e-8 absolute, final state fidelity 1 - F <= 1e-10 (north star),
Krylov iterations within 1 (the fused path uses the plain three-term recurrence), sample counts exact
(the same PCG64 draws on a state equal to 1e-10)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def _program(rs, d):
    kinds = {"Constant": lambda s: rs.Constant(s["duration_ns"], s["value"]),
             "Ramp": lambda s: rs.Ramp(s["duration_ns"], s["start"], s["stop"]),
             "Blackman": lambda s: rs.Blackman(s["duration_ns"], s["area"])}
    om = [[kinds[s["kind"]](s) for s in ch] for ch in d["omega"]]
    de = [[kinds[s["kind"]](s) for s in ch] for ch in d["delta"]]
    return rs.ChannelProgram.from_channels(om, de, d["duration_ns"])


def _config(rs, runner, c):
    specs = tuple(rs.ObservableSpec(k, tuple(q), e) for k, q, e in c["observables"])
    return runner.RunConfig(dt_ns=c["dt_ns"], krylov=rs.KrylovConfig(c["tolerance"], c["max_krylov_dim"]),
                            observables=specs, snapshot_every=c["snapshot_every"], initial_bits=c["initial_bits"],
                            seed=c["seed"], sample_shots=c["sample_shots"])


def test_config_validation_and_document_roundtrip(tmp_path):
    import paper_2510_09813_b200 as rs
    from paper_2510_09813_b200 import runner

    with pytest.raises(rs.ValidationError):
        runner.RunConfig(backend="gpu")
    with pytest.raises(rs.ValidationError):
        runner.RunConfig(dt_ns=0)
    with pytest.raises(rs.ValidationError):
        runner.RunConfig(sample_shots=-1)
    cfg = runner.RunConfig(seed=3, sample_shots=10)
    assert cfg.echo()["krylov"]["tolerance"] == 1e-10 and cfg.echo()["sample_shots"] == 10
    doc = {"metadata": {"timestamp_utc": "x", "qubit_count": 2}, "observables": [],
           "diagnostics": {"total_wall_time_s": 1.0, "wall_time_per_step_s": [0.5], "krylov_iterations": [3]},
           "final_state": {"re": [1.0, 0.0], "im": [0.0, 0.0]}, "snapshots": [], "samples": None}
    res = runner.RunResult(doc)
    res.save(tmp_path / "out" / "r.json")
    back = runner.RunResult.load(tmp_path / "out" / "r.json")
    assert back == res and np.array_equal(back.final_state, [1.0, 0.0])
    stripped = back.strip_volatile()
    assert "timestamp_utc" not in stripped["metadata"] and stripped["diagnostics"] == {"krylov_iterations": [3]}
    assert not any(p.name.endswith(".tmp") for p in (tmp_path / "out").iterdir())


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["adiabatic5", "adiabatic5_var"])
def test_execute_run_matches_reference(case):
    import paper_2510_09813_b200 as rs
    from paper_2510_09813_b200 import runner

    g = json.load(open(os.path.join(GOLDEN, "runs_sv.json")))[case]
    ref = g["document"]
    reg = rs.Register(tuple(map(tuple, g["register"]["positions_um"])), g["register"]["interaction_c"])
    res = runner.execute_run(reg, _program(rs, g["program"]), _config(rs, runner, g["config"]))
    doc = res.strip_volatile()
    for key in ("qubit_count", "dt_ns", "duration_ns", "step_count"):
        assert doc["metadata"][key] == ref["metadata"][key]
    assert len(doc["observables"]) == len(ref["observables"])
    for a, b in zip(doc["observables"], ref["observables"]):
        assert (a["spec_index"], a["kind"], a["qubits"], a["step"], a["t_ns"]) == \
               (b["spec_index"], b["kind"], b["qubits"], b["step"], b["t_ns"])
        assert np.abs(np.array(a["values"]) - np.array(b["values"])).max() <= 1e-8
    it_a = np.array(doc["diagnostics"]["krylov_iterations"])
    it_b = np.array(ref["diagnostics"]["krylov_iterations"])
    assert np.abs(it_a - it_b).max() <= 1
    psi = res.final_state
    ref_psi = np.asarray(ref["final_state"]["re"]) + 1j * np.asarray(ref["final_state"]["im"])
    assert 1.0 - abs(np.vdot(ref_psi, psi)) ** 2 <= 1e-10
    assert len(doc["snapshots"]) == len(ref["snapshots"])
    for a, b in zip(doc["snapshots"], ref["snapshots"]):
        assert a["t_ns"] == b["t_ns"]
        assert np.abs(np.array(a["re"]) + 1j * np.array(a["im"]) - np.array(b["re"]) - 1j * np.array(b["im"])).max() <= 1e-8
    assert doc["samples"] == ref["samples"]


def test_foreign_observable_specs_are_accepted():
    # rydsim's ObservableSpec objects (or anything with its fields) pass through evolve_sv unchanged
    from types import SimpleNamespace

    import paper_2510_09813_b200 as rs
    from paper_2510_09813_b200.sv import as_spec

    spec = as_spec(SimpleNamespace(kind="correlation", qubits=[0, 1, 2, 3], every_n_steps=0))
    assert isinstance(spec, rs.ObservableSpec) and spec.qubits == (0, 1, 2, 3) and spec.every_n_steps == 0
    mine = rs.ObservableSpec("occupation", (1,), 2)
    assert as_spec(mine) is mine
    with pytest.raises(rs.ValidationError):
        as_spec(SimpleNamespace(kind="entropy", qubits=(), every_n_steps=1))
