"""Where the time of evolve_sv goes on a small register (configs[1], N=20): engine set-up, the steps,
the final copy. usage: python tools/e2e_breakdown.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_09813_b200 as rs  # noqa: E402
from paper_2510_09813_b200 import workloads  # noqa: E402
from paper_2510_09813_b200.engine import SvEngine  # noqa: E402

reg, seq = workloads.config("lattice20")
u = rs.interaction_matrix(reg)
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = SvEngine(20, u, max_krylov_dim=100)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng.close()
    del eng
    torch.cuda.synchronize()
    host_in = torch.zeros(2 ** 20, dtype=torch.complex128, pin_memory=True)
    host_in[0] = 1.0
    t2 = time.perf_counter()
    res = rs.evolve_sv(seq, reg, rs.SvRunConfig(krylov=rs.KrylovConfig(1e-10), initial_state=host_in,
                                                observables=(rs.ObservableSpec("occupation", (), 1),)))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out[rep] = {"engine_setup_ms": 1e3 * (t1 - t0), "evolve_sv_ms": 1e3 * (t3 - t2),
                "steps_wall_ms": 1e3 * sum(res.step_wall_times_s)}
    del res
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
