"""configs[1] (N=20) step loop: device-timed wall of 297 steps with and without the per-kernel
profiling events, GPU busy fraction (profiled kernel time / wall). usage: python tools/l20_overhead.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_09813_b200 import interaction_matrix, workloads  # noqa: E402
from paper_2510_09813_b200.engine import SvEngine  # noqa: E402

reg, seq = workloads.config("lattice20")
out = {}
for prof in (False, True, False, True):
    eng = SvEngine(20, interaction_matrix(reg), max_krylov_dim=100)
    eng.set_observables([1 << q for q in range(20)])
    for k in range(3):
        eng.step(*seq.step(k), float(seq.dt_ns), 1e-10, 100, next_params=seq.step(k + 1), observe=True)
        eng.observables()
    eng.set_profiling(prof)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    t0 = time.perf_counter()
    host_step = 0.0
    mv = 0
    for k in range(3, 300):
        nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
        h0 = time.perf_counter()
        rep = eng.step(*seq.step(k), float(seq.dt_ns), 1e-10, 100, next_params=nxt, observe=True)
        host_step += time.perf_counter() - h0
        eng.observables()
        mv += rep.matvecs
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    row = {"ms": ms, "wall_ms": 1e3 * (time.perf_counter() - t0), "in_step_ms": 1e3 * host_step, "matvecs": mv,
           "hpsi_s": mv / (ms / 1e3)}
    if prof:
        p = eng.profile()
        row["kernel_ms"] = {f: v["ms"] for f, v in p.items()}
        row["busy"] = sum(v["ms"] for v in p.values()) / ms
    out[f"profiling={prof}#{len(out)}"] = row
    del eng
print(json.dumps(out, indent=1))
