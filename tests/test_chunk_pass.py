"""GPU parity of the L2-resident chunk pass (rsv::ChunkArgs, opt-in through rsv_set_plan): the
first kernel of a Lanczos iteration, which applies two bit groups (L tiles: bits [0, 12); M tiles: bits
[12, 12 + gm)) with one HBM round trip. The plan override forces it at small N too, so it
is checked against the CPU oracle (reference hamiltonian.py:164 / sv.py:80 restated in
oracle/sv_oracle.py) on the same seeded inputs:

* H.psi: relative 1e-12 of max |H psi| (as the reference's hamiltonian tests);
* evolution: fidelity 1 - |<ref|gpu>|^2 <= 1e-10, occupations within 1e-8 (north-star bar);
* scheduler: every lag (L tiles right behind their chunk, or all M tiles first) gives the same
  bits, and back-to-back launches reuse the reset ticket/counters.
"""

import numpy as np
import pytest

from oracle import sv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


def random_slice(rng, n):
    om = rng.uniform(0.0, 4.0, n)
    de = rng.uniform(-3.0, 3.0, n)
    u = np.triu(rng.uniform(0.0, 2.0, (n, n)), 1)
    return om, de, u + u.T


def rel_err(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


def apply_with_plan(torch, n, om, de, u, psi, gm, lag=-1, diag="fly"):
    from paper_2510_09813_b200 import _native as nat
    from paper_2510_09813_b200.engine import Context

    ctx = Context(n, u if diag == "fly" else np.zeros((n, n)), diag=diag)
    ctx.set_plan(gm, lag)
    plan = ctx.pass_plan()
    x = torch.from_numpy(psi).cuda()
    y = torch.empty_like(x)
    dvec = None
    if diag == "vec":
        dvec = torch.from_numpy(O.build_diagonal(de, u)).cuda()
        de = np.zeros(n)
    ctx.sync_stream()
    if dvec is not None:
        nat.check(ctx.lib.rsv_bind_diag_vector(ctx.ctx, dvec.data_ptr(), 0))
    nat.check(ctx.lib.rsv_apply_hamiltonian(ctx.ctx, nat.dptr(np.ascontiguousarray(om)),
                                            nat.dptr(np.ascontiguousarray(de)), x.data_ptr(), y.data_ptr()))
    out = y.cpu().numpy()
    ctx.close()
    return out, plan


@pytest.mark.parametrize("n,gm", [(16, 3), (17, 4), (18, 5), (19, 6), (20, 7), (21, 8), (22, 9), (22, 8),
                                  (23, 8)])
def test_apply_against_oracle(torch, n, gm):
    rng = np.random.default_rng(100 + n + gm)
    om, de, u = random_slice(rng, n)
    om[(3 * n) // 4] = 0.0   # zero drives are skipped (_kernels.py:19)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
    out, plan = apply_with_plan(torch, n, om, de, u, psi, gm)
    assert plan[0]["family"] == "chunk"
    assert plan[0]["chunk_bits"] == 12 + gm
    assert rel_err(out, ref) <= 1e-12


@pytest.mark.parametrize("lag", [8, 12, 32, 1 << 20])
def test_scheduler_lag_is_bit_exact(torch, lag):
    # gm = 3: 8 tiles of each kind per chunk; lag 8 puts each chunk's first L tile right
    # behind its last M tile, 2^20 (clamped to the tile count) hands out every M tile first
    n = 18
    rng = np.random.default_rng(7)
    om, de, u = random_slice(rng, n)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    base, _ = apply_with_plan(torch, n, om, de, u, psi, 3, 12)
    out, _ = apply_with_plan(torch, n, om, de, u, psi, 3, lag)
    assert np.array_equal(out, base)
    ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
    assert rel_err(out, ref) <= 1e-12


def test_vec_diagonal(torch):
    n = 18
    rng = np.random.default_rng(11)
    om, de, u = random_slice(rng, n)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    ref = O.apply_hamiltonian(om, O.build_diagonal(de, u), psi)
    out, plan = apply_with_plan(torch, n, om, de, u, psi, 4, diag="vec")
    assert plan[0]["family"] == "chunk"
    assert rel_err(out, ref) <= 1e-12


def test_plan_override_errors():
    from paper_2510_09813_b200 import _native as nat
    from paper_2510_09813_b200.engine import Context

    ctx = Context(16, np.zeros((16, 16)))
    with pytest.raises(Exception):
        ctx.set_plan(2)          # M tiles need >= 3 group bits
    with pytest.raises(Exception):
        ctx.set_plan(4 + 1)      # 12 + 5 > 16 - 1: no hi pass left
    ctx.set_plan(0)
    assert all(p["family"] != "chunk" for p in ctx.pass_plan())
    ctx.set_plan(-1)             # auto: plain passes (the chunk pass is opt-in); at 16..21 qubits the
    plan = ctx.pass_plan()       # lo and last passes run fused in one launch (iter2)
    assert plan[0]["family"] in ("lo", "iter2") and plan[0]["lo"]
    assert all(p["family"] != "chunk" for p in plan)
    assert isinstance(nat.RSV_DIAG_FLY, int)
    ctx.close()


@pytest.mark.parametrize("gm,diag", [(3, "fly"), (4, "vec")])
def test_evolution_against_oracle(gm, diag):
    from paper_2510_09813_b200 import interaction_matrix, workloads
    from paper_2510_09813_b200.engine import SvEngine

    n = 17
    reg, seq = workloads.config("random29", n_override=n)
    u = interaction_matrix(reg)
    steps = list(range(30, 42))   # mid-pulse: strong drive, ~20 Krylov vectors per step
    om = np.array([seq.step(k)[0] for k in steps])
    de = np.array([seq.step(k)[1] for k in steps])
    eng = SvEngine(n, u, diag=diag, max_krylov_dim=100)
    eng.set_plan(gm)
    assert eng.pass_plan()[0]["family"] == "chunk"
    eng.set_observables([1 << q for q in range(n)])
    for i in range(len(steps)):
        nxt = (om[i + 1], de[i + 1]) if i + 1 < len(steps) else None
        rep = eng.step(om[i], de[i], 10.0, 1e-10, 100, next_params=nxt, observe=True)
        assert rep.converged
    psi = eng.state().cpu().numpy()
    occ = eng.observables()
    ref = O.evolve_sv(om, de, 10.0, u, tolerance=1e-10, observe_every=0)
    fid = abs(np.vdot(ref["final_state"], psi)) ** 2
    assert 1.0 - fid <= 1e-10
    assert np.abs(occ - ref["occupations"][-1][2]).max() <= 1e-8
    eng.close()
