"""Full-size parity of the fused Lanczos step (GPU box): the whole N=29 1 us pulse of bench.py run
twice -- the fused three-term recurrence (the product default) and the reference's algorithm with
full re-orthogonalisation of every Lanczos vector (krylov.py:103-104, KrylovConfig(reorthogonalize=
True)) -- and compared: fidelity 1 - |<a|b>|^2, max |occupation difference|, energies, Krylov counts.

usage: python tools/full_pulse_parity.py [N] [steps]  -> JSON line
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_09813_b200 import interaction_matrix, overlap, workloads  # noqa: E402
from paper_2510_09813_b200.engine import SvEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 29
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reg, seq = workloads.config("random29", n_override=n)
u = interaction_matrix(reg)


def run(reorth):
    eng = SvEngine(n, u, diag="fly", max_krylov_dim=100)
    eng.set_reorthogonalize(reorth)
    eng.set_observables([1 << q for q in range(n)])
    t0 = time.time()
    mv, energies = 0, []
    for k in range(steps):
        nxt = seq.step(k + 1) if k + 1 < steps else None
        rep = eng.step(*seq.step(k), float(seq.dt_ns), 1e-10, 100, next_params=nxt, observe=(k + 1 == steps))
        assert rep.converged, k
        mv += rep.matvecs
        energies.append(rep.alpha0)
    occ = eng.observables()
    torch.cuda.synchronize()
    return eng, occ, mv, np.array(energies), time.time() - t0


eng_a, occ_a, mv_a, e_a, t_a = run(False)
host = torch.empty(2 ** n, dtype=torch.complex128, pin_memory=True)
host.copy_(eng_a.state())
eng_a.close()
del eng_a
torch.cuda.empty_cache()
eng_b, occ_b, mv_b, e_b, t_b = run(True)
other = eng_b.slots[1]   # free after the run
other.copy_(host)
ov = overlap(other, eng_b.state())
line = {"n": n, "steps": steps, "fidelity_defect": 1.0 - abs(ov) ** 2,
        "max_occupation_diff": float(np.abs(occ_a - occ_b).max()),
        "max_energy_diff": float(np.abs(e_a - e_b).max()),
        "matvecs": {"three_term": mv_a, "reorthogonalized": mv_b},
        "wall_s": {"three_term": round(t_a, 1), "reorthogonalized": round(t_b, 1)}}
print(json.dumps(line))
