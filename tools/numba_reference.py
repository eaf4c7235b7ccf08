"""Build container only: the REAL reference kernel (rydsim/_kernels.py:13, imported from
/root/reference) against its restatement oracle/numba_ref.py -- identical outputs, same time per
element -- so the GPU box's numba timing (bench.py --impl reference, 'reference_numba') stands for
the reference's own CPU kernel. Writes profiles/r2_numba_reference.json.

usage: python tools/numba_reference.py [N]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
from rydsim._kernels import matvec_bitflip_diag  # noqa: E402

from oracle.numba_ref import matvec_bitflip_diag_range  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
rng = np.random.default_rng(1)
dim = 1 << n
psi = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
diag = rng.uniform(-10, 10, dim)
half = 0.5 * rng.uniform(0.5, 4.0, n)
half[3] = 0.0
a = np.empty_like(psi)
b = np.empty_like(psi)
matvec_bitflip_diag(psi[:1024].copy(), diag[:1024].copy(), half[:10].copy(), a[:1024])   # compile
matvec_bitflip_diag_range(psi, diag, half, b, 0, 64)
reps = 3
t = []
for _ in range(reps):
    t0 = time.perf_counter()
    matvec_bitflip_diag(psi, diag, half, a)
    t.append(time.perf_counter() - t0)
t2 = []
for _ in range(reps):
    t0 = time.perf_counter()
    matvec_bitflip_diag_range(psi, diag, half, b, 0, dim)
    t2.append(time.perf_counter() - t0)
same = bool(np.array_equal(a, b))
out = {"n": n, "identical_outputs": same, "reference_kernel_s": min(t), "restatement_s": min(t2),
       "ratio": min(t2) / min(t), "reference_hpsi_per_s": 1.0 / min(t),
       "host": os.uname().nodename, "cores_used": 1,
       "note": "rydsim/_kernels.py:13 imported from /root/reference (build container) vs oracle/numba_ref.py"}
print(json.dumps(out))
with open(os.path.join(ROOT, "profiles", "r2_numba_reference.json"), "w") as fh:
    json.dump(out, fh, indent=1)
