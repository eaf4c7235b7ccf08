"""Run orchestration for the state-vector backend -- mirror of rydsim/runner.py (``execute_run``,
``RunResult``, ``write_json_atomic``; runner.py:1-357) and of the run knobs of
rydsim/sequence_io.py:142 ``RunConfig``.

``execute_run(register, program, cfg)`` samples and discretizes the program (pulses.py), runs
``evolve_sv`` on the B200 path, samples bitstrings on the device and packages the same
JSON-serializable document as the reference (metadata / observables / diagnostics / final_state /
snapshots / samples), so reference tooling that reads result files keeps working. Only the
``"sv"`` backend is on this path; ``"mps"`` and ``"oracle"`` are out of scope and are
rejected with a ValidationError naming the reference package that still provides them.
"""

from __future__ import annotations

import hashlib
import json
import os
import tempfile
import time
from dataclasses import dataclass, field
from datetime import datetime, timezone
from pathlib import Path

import numpy as np

from . import __version__
from .errors import ValidationError
from .krylov import KrylovConfig
from .observables import ObservableSpec, format_bitstring, sample_bitstrings
from .pulses import discretize, sample_program
from .sv import SvRunConfig, evolve_sv

__all__ = ["RunConfig", "RunResult", "execute_run", "write_json_atomic", "VOLATILE_FIELDS",
           "DENSE_CONVERSION_CAP"]

# runner.py:40-44: fields that legitimately differ between identical runs (timing only)
VOLATILE_FIELDS = (
    ("metadata", "timestamp_utc"),
    ("diagnostics", "wall_time_per_step_s"),
    ("diagnostics", "total_wall_time_s"),
)
DENSE_CONVERSION_CAP = 20   # rydsim/mps/state.py: final states are stored for N <= 20 by default


@dataclass(frozen=True)
class RunConfig:
    """sequence_io.py:142 RunConfig (the fields a state-vector run reads)."""

    backend: str = "sv"
    dt_ns: int = 10
    krylov: KrylovConfig = field(default_factory=KrylovConfig)
    observables: tuple = (ObservableSpec("occupation", (), 1),)
    snapshot_every: int = 0
    store_final_state: bool | None = None   # None = auto (N <= 20)
    initial_bits: int = 0
    seed: int = 0
    sample_shots: int = 0
    threads: int | None = None
    memory_budget_bytes: int | None = None
    qubit_cap: int = 30
    allow_above_cap: bool = False
    output: str | None = None

    def __post_init__(self):
        if self.backend not in ("sv", "mps", "oracle"):
            raise ValidationError(f"backend must be sv, mps or oracle, got {self.backend!r}")
        if self.dt_ns < 1:
            raise ValidationError(f"dt_ns must be >= 1, got {self.dt_ns}")
        if self.sample_shots < 0 or self.snapshot_every < 0:
            raise ValidationError("sample_shots and snapshot_every must be >= 0")

    def echo(self) -> dict:
        """The knob dump of the result metadata (sequence_io.py:175, state-vector knobs)."""
        return {
            "backend": self.backend,
            "dt_ns": self.dt_ns,
            "krylov": {"tolerance": self.krylov.tolerance, "max_krylov_dim": self.krylov.max_krylov_dim,
                       "norm_epsilon": self.krylov.norm_epsilon},
            "observables": [{"type": s.kind, "qubits": list(s.qubits), "every_n_steps": s.every_n_steps}
                            for s in self.observables],
            "snapshot_every": self.snapshot_every,
            "store_final_state": self.store_final_state,
            "initial_bits": self.initial_bits,
            "seed": self.seed,
            "sample_shots": self.sample_shots,
            "threads": self.threads,
            "memory_budget_bytes": self.memory_budget_bytes,
            "qubit_cap": self.qubit_cap,
            "allow_above_cap": self.allow_above_cap,
        }


def _native(obj):
    """runner.py:50: numpy scalars/arrays -> JSON-native values."""
    if isinstance(obj, dict):
        return {k: _native(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_native(v) for v in obj]
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.floating):
        return float(obj)
    if isinstance(obj, np.ndarray):
        return [_native(v) for v in obj.tolist()]
    if isinstance(obj, np.bool_):
        return bool(obj)
    return obj


def _host(state) -> np.ndarray:
    if hasattr(state, "detach"):
        return state.detach().cpu().numpy()
    return np.asarray(state)


def _state_payload(state) -> dict:
    s = _host(state)
    return {"re": [float(x) for x in s.real], "im": [float(x) for x in s.imag]}


def _state_from_payload(payload) -> np.ndarray:
    return np.asarray(payload["re"]) + 1j * np.asarray(payload["im"])


class RunResult:
    """runner.py:78: thin wrapper over the serialized result document."""

    def __init__(self, data: dict):
        self.data = data

    def __eq__(self, other):
        return isinstance(other, RunResult) and self.data == other.data

    @property
    def metadata(self) -> dict:
        return self.data["metadata"]

    @property
    def observables(self) -> list:
        return self.data["observables"]

    @property
    def diagnostics(self) -> dict:
        return self.data["diagnostics"]

    @property
    def final_state(self):
        payload = self.data.get("final_state")
        return None if payload is None else _state_from_payload(payload)

    @property
    def snapshots(self):
        return [(s["t_ns"], _state_from_payload(s)) for s in self.data.get("snapshots", [])]

    def to_json(self) -> str:
        return json.dumps(self.data, indent=1)

    @classmethod
    def from_json(cls, text: str) -> "RunResult":
        return cls(json.loads(text))

    def save(self, path):
        write_json_atomic(path, self.to_json())

    @classmethod
    def load(cls, path) -> "RunResult":
        return cls.from_json(Path(path).read_text())

    def strip_volatile(self) -> dict:
        doc = json.loads(self.to_json())
        for section, key in VOLATILE_FIELDS:
            doc.get(section, {}).pop(key, None)
        return doc


def write_json_atomic(path, text: str):
    """runner.py:138: temp file + rename, so a failure never leaves a partial output."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=f".{path.name}.", suffix=".tmp")
    try:
        with os.fdopen(fd, "w") as handle:
            handle.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _sequence_digest(register, program) -> str:
    return hashlib.sha256(repr((register, program)).encode()).hexdigest()[:16]


def execute_run(register, program, cfg: RunConfig = RunConfig()) -> RunResult:
    """runner.py:179 execute_run for backend "sv": discretize, evolve on the GPU, sample, package."""
    if cfg.backend != "sv":
        raise ValidationError(f"backend {cfg.backend!r} is not on the B200 path (only 'sv'); "
                              "run it with the reference package rydsim")
    n = register.qubit_count
    seq = discretize(sample_program(program), cfg.dt_ns)
    if seq.qubit_count != n:
        raise ValidationError(f"program has {seq.qubit_count} channels but register has {n} atoms")
    store_final = cfg.store_final_state
    if store_final is None:
        store_final = n <= DENSE_CONVERSION_CAP
    elif store_final and n > DENSE_CONVERSION_CAP:
        raise ValidationError(f"dense final-state artifacts need N <= {DENSE_CONVERSION_CAP}")

    started = time.perf_counter()
    initial = None
    if cfg.initial_bits:
        initial = np.zeros(2 ** n, dtype=complex)
        initial[cfg.initial_bits] = 1.0
    res = evolve_sv(seq, register, SvRunConfig(
        krylov=cfg.krylov, initial_state=initial, observables=tuple(cfg.observables),
        snapshot_every=cfg.snapshot_every, qubit_cap=cfg.qubit_cap, allow_above_cap=cfg.allow_above_cap,
        memory_budget_bytes=cfg.memory_budget_bytes))
    samples = None
    if cfg.sample_shots:
        indices = sample_bitstrings(res.final_state, cfg.sample_shots, cfg.seed)   # on the device
        counts: dict[str, int] = {}
        for b in indices:
            key = format_bitstring(int(b), n)
            counts[key] = counts.get(key, 0) + 1
        samples = {"shots": cfg.sample_shots, "seed": cfg.seed, "counts": dict(sorted(counts.items()))}
    total_wall = time.perf_counter() - started

    metadata = {
        "tool": "paper_2510_09813_b200",
        "version": __version__,
        "numpy_version": np.__version__,
        "timestamp_utc": datetime.now(timezone.utc).isoformat(),
        "backend": cfg.backend,
        "device": "cuda (B200 bit-group passes)",
        "qubit_count": n,
        "dt_ns": seq.dt_ns,
        "duration_ns": seq.duration_ns,
        "step_count": seq.step_count,
        "sequence_digest": _sequence_digest(register, program),
        "config": cfg.echo(),
    }
    observables = [{"spec_index": r.spec_index, "kind": r.kind, "qubits": list(r.qubits), "step": r.step,
                    "t_ns": float(r.t_ns), "values": [float(v) for v in r.values]} for r in res.observables]
    diagnostics = {
        "peak_memory_bytes": res.peak_memory_bytes,
        "krylov_iterations": [r.iterations for r in res.krylov_reports],
        "krylov_residuals": [float(r.residual) for r in res.krylov_reports],
        "wall_time_per_step_s": [float(t) for t in res.step_wall_times_s],
        "total_wall_time_s": float(total_wall),
    }
    doc = {
        "metadata": metadata,
        "observables": observables,
        "diagnostics": diagnostics,
        "final_state": _state_payload(res.final_state) if store_final else None,
        "snapshots": [{"t_ns": float(t), **_state_payload(s)} for t, s in res.snapshots],
        "samples": samples,
    }
    return RunResult(_native(doc))
