"""Debug: apply_hamiltonian vs the oracle at several N; reports where the result differs (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_09813_b200 as rs  # noqa: E402
from oracle import sv_oracle as O  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [20, 21, 22, 23]:
    rng = np.random.default_rng(n)
    om = rng.uniform(0.5, 3.0, n)
    de = rng.uniform(-2, 2, n)
    pos = rng.uniform(0, 30, (n, 2))
    d = np.linalg.norm(pos[:, None] - pos[None], axis=-1) + np.eye(n)
    u = 100.0 / d ** 6
    np.fill_diagonal(u, 0.0)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
    s = rs.HamiltonianSlice.from_parameters(om, de, u)
    out = rs.apply_hamiltonian(s, torch.from_numpy(psi).cuda()).cpu().numpy()
    err = np.abs(out - ref)
    bad = np.nonzero(err > 1e-9 * np.abs(ref).max())[0]
    print(n, os.environ.get("RSV_LIB", "default"), "rel", float(np.linalg.norm(out - ref) / np.linalg.norm(ref)),
          "bad", len(bad), "first", bad[:8].tolist(), "bits", [int(b).bit_length() for b in bad[:4]], flush=True)
