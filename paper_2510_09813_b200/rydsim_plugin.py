"""The reference-side switch: route rydsim's state-vector backend through the B200 path.

This is the change INTEGRATION.md describes for rydsim/sv.py:80 (``evolve_sv``), packaged so it
can be installed without editing the reference (``install()``) and exercised by tests with the
real rydsim objects. With ``RYDSIM_DEVICE=b200`` in the environment (or ``install(force=True)``)
``rydsim.sv.evolve_sv`` -- and the name rydsim's run harness bound at import
(rydsim/runner.py:34, called at :206 for backend "sv") -- run ``paper_2510_09813_b200.evolve_sv``:

* arguments: rydsim's ``DiscretizedSequence``, ``Register``, ``SvRunConfig`` (krylov,
  initial_state, observables, snapshot_every, qubit_cap, allow_above_cap, memory_budget_bytes,
  force_numpy_matvec) are passed through unchanged (the B200 path reads the same fields);
* result: rydsim's own ``SvRunResult`` (sv.py:64) with numpy ``final_state`` and snapshots,
  rydsim ``ObservableRecord`` (observables.py:263) and ``KrylovReport`` (krylov.py:48) objects;
* errors: this package's exceptions derive from rydsim's when rydsim is importable
  (errors.py), so rydsim/cli.py:248-258 maps them to the same exit codes.

Everything else in rydsim (MPS backend, CLI, configs, run documents) is untouched.
"""

from __future__ import annotations

import os

__all__ = ["install", "uninstall", "evolve_sv_b200", "DEVICE_ENV"]

DEVICE_ENV = "RYDSIM_DEVICE"
_saved = {}


def _reference_modules():
    import rydsim.krylov as rk
    import rydsim.observables as ro
    import rydsim.sv as rsv

    return rsv, ro, rk


def evolve_sv_b200(seq, reg, cfg=None):
    """rydsim.sv.evolve_sv (sv.py:80) on the B200: same arguments, rydsim's result types."""
    from . import sv as b200_sv

    rsv, ro, rk = _reference_modules()
    if cfg is None:
        cfg = rsv.SvRunConfig()
    b_cfg = b200_sv.SvRunConfig(
        krylov=cfg.krylov,
        initial_state=cfg.initial_state,
        observables=tuple(cfg.observables),
        snapshot_every=cfg.snapshot_every,
        qubit_cap=cfg.qubit_cap,
        allow_above_cap=cfg.allow_above_cap,
        memory_budget_bytes=cfg.memory_budget_bytes,
        force_numpy_matvec=getattr(cfg, "force_numpy_matvec", False),
        host_final_state=True,
    )
    res = b200_sv.evolve_sv(seq, reg, b_cfg)
    records = [ro.ObservableRecord(r.spec_index, r.kind, tuple(r.qubits), r.step, r.t_ns, list(r.values))
               for r in res.observables]
    reports = [rk.KrylovReport(iterations=r.iterations, converged=r.converged, residual=r.residual)
               for r in res.krylov_reports]
    return rsv.SvRunResult(
        final_state=res.final_state,
        observables=records,
        krylov_reports=reports,
        step_wall_times_s=list(res.step_wall_times_s),
        peak_memory_bytes=res.peak_memory_bytes,
        snapshots=list(res.snapshots),
        dt_ns=res.dt_ns,
        duration_ns=res.duration_ns,
    )


def install(force: bool = False):
    """Patch rydsim.sv.evolve_sv (and rydsim.runner's binding of it) with the device switch."""
    import rydsim.runner as rr
    import rydsim.sv as rsv

    if "sv" in _saved:
        return
    original = rsv.evolve_sv
    _saved["sv"] = original
    _saved["runner"] = rr.evolve_sv

    def evolve_sv(seq, reg, cfg=rsv.SvRunConfig()):
        if force or os.environ.get(DEVICE_ENV, "").lower() == "b200":
            return evolve_sv_b200(seq, reg, cfg)
        return original(seq, reg, cfg)

    evolve_sv.__doc__ = original.__doc__
    evolve_sv.__wrapped__ = original
    rsv.evolve_sv = evolve_sv
    rr.evolve_sv = evolve_sv


def uninstall():
    import rydsim.runner as rr
    import rydsim.sv as rsv

    if "sv" in _saved:
        rsv.evolve_sv = _saved.pop("sv")
        rr.evolve_sv = _saved.pop("runner")
