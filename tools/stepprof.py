"""Per-step Krylov dimension, regenerated vectors, splits and per-family kernel time (GPU box).

usage: python tools/stepprof.py N STEPS [regen=1] [cap=-1] [spec=-1] [first=0]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_09813_b200 import interaction_matrix, workloads  # noqa: E402
from paper_2510_09813_b200.engine import SvEngine  # noqa: E402

n = int(sys.argv[1])
steps = int(sys.argv[2])
regen = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cap = int(sys.argv[4]) if len(sys.argv) > 4 else -1
spec = int(sys.argv[5]) if len(sys.argv) > 5 else -1
first = int(sys.argv[6]) if len(sys.argv) > 6 else 0
reg, seq = workloads.config("random29" if n >= 21 else "lattice20", n_override=n if n >= 21 else None)
eng = SvEngine(n, interaction_matrix(reg), max_krylov_dim=100, krylov_vectors_cap=None if cap < 0 else cap)
eng.set_tail_regeneration(bool(regen))
eng.set_speculation(spec)
eng.set_observables([1 << q for q in range(n)])
for k in range(first):
    eng.step(*seq.step(k), float(seq.dt_ns), 1e-10, 100, next_params=seq.step(k + 1))
eng.set_profiling(True)
tot = {"lo": 0, "mid": 0, "last": 0, "combine": 0}
rows = []
prev = {f: (0.0, 0) for f in tot}
for k in range(first, first + steps):
    nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
    r = eng.step(*seq.step(k), float(seq.dt_ns), 1e-10, 100, next_params=nxt, observe=True)
    eng.observables()
    p = eng.profile()
    row = {"step": k, "k": r.iterations, "regen": r.regenerated, "split": r.substeps, "mv": r.matvecs}
    for f, v in p.items():
        key = "lo" if f in ("lo", "first", "chunk", "iter2") else f
        d_ms = v["ms"] - prev[key][0]
        d_n = v["launches"] - prev[key][1]
        prev[key] = (v["ms"], v["launches"])
        row[key] = [round(d_ms, 2), d_n]
    rows.append(row)
    print(json.dumps(row), flush=True)
print(json.dumps({"n": n, "regen": regen, "cap": eng.krylov_cap, "matvecs": sum(r["mv"] for r in rows),
                  "ms": {f: round(sum(r[f][0] for r in rows if f in r), 1) for f in tot}}))
