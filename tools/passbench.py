"""Per-kernel-family bandwidth of the Lanczos step at size N (quick A/B tool, GPU box only).

usage: RSV_LIB=tools/_rsv_x.so python tools/passbench.py N [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_09813_b200 import interaction_matrix, workloads  # noqa: E402
from paper_2510_09813_b200.engine import SvEngine  # noqa: E402

n = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reg, seq = workloads.config("random29", n_override=n)
eng = SvEngine(n, interaction_matrix(reg), diag=os.environ.get("RSV_DIAG", "fly"), max_krylov_dim=100)
eng.set_plan(int(os.environ.get("RSV_PLAN_GM", "-1")), int(os.environ.get("RSV_PLAN_LAG", "-1")))
for k in range(3):
    eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1))
eng.set_profiling(True)
mv = 0
for k in range(3, 3 + steps):
    r = eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1))
    mv += r.matvecs
prof = eng.profile()
amp = 2 ** n
alg = {"lo": 48 * amp, "first": 48 * amp, "chunk": 48 * amp, "mid": 48 * amp, "last": 48 * amp, "iter2": 96 * amp}   # x + elementwise operand + out
out = {"lib": os.environ.get("RSV_LIB", "default"), "n": n, "matvecs": mv, "gm": os.environ.get("RSV_PLAN_GM", "-1"), "lag": os.environ.get("RSV_PLAN_LAG", "-1")}
for f, v in prof.items():
    if v["launches"] and f in alg:
        ms = v["ms"] / v["launches"]
        out[f] = {"ms": round(ms, 3), "GBps": round(alg[f] / ms / 1e6)}
    elif v["launches"]:
        out[f] = {"ms": round(v["ms"] / v["launches"], 3)}
tot = sum(v["ms"] for v in prof.values())
out["eff_GBps_per_hpsi"] = round(mv * 32 * amp / (tot / 1e3) / 1e9)
print(json.dumps(out))
