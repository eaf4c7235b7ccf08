"""Parity at the headline sizes: the CUDA path against the reference's algorithm on the host.

BASELINE configs[2] (N=27 3x9 lattice) and configs[3] (N=29 random register with a detuning map)
are the sizes the speed-up is quoted on, and N=29/30 are the only sizes whose pass plans use a
9-bit strided group (5-D tensor map with a non-trivial second group dimension; at N=29 it is the
mid pass that also takes over qubits 0..2). These tests compare, on the same GPU-produced
mid-pulse states:

* one H.psi over the WHOLE output vector with the C restatement of the reference's compiled
  matvec (oracle/sv_ref.c svref_matvec = rydsim/_kernels.py:13), relative error <= 1e-12 of
  max |H psi| (the reference's hamiltonian tests use 1e-12), reported per output slice so both
  ends of the index and the slices that cross group boundaries are named on failure;
* whole Lanczos steps with the reference's algorithm (full re-orthogonalisation,
  rydsim/krylov.py:67-125, oracle/big.py) driven by that matvec: fidelity
  1 - |<psi_ref|psi_gpu>|^2 <= 1e-10, occupations and energy (= alpha_0) within 1e-8
  absolute (north-star acceptance), Krylov iteration counts within one.

Host memory: the N=29 step keeps the reference's whole basis on the host (16 vectors of
8.6 GB at the step used here; the GPU box has 196 GB).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rs():
    import paper_2510_09813_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


def _mid_pulse_state(rs, torch, name, n, steps, cap, n_override=None):
    """Evolve |0..0> through `steps` steps of a workload on the GPU; return (reg, seq, u, host state)."""
    from paper_2510_09813_b200 import workloads
    from paper_2510_09813_b200.engine import SvEngine

    reg, seq = workloads.config(name, n_override=n_override)
    u = rs.interaction_matrix(reg)
    eng = SvEngine(n, u, diag="fly", max_krylov_dim=100, krylov_vectors_cap=cap)
    try:
        for k in range(steps):
            rep = eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=seq.step(k + 1))
            assert rep.converged
        host = eng.state().cpu().numpy()
    finally:
        eng.close()
        eng.slots = []
        del eng
        torch.cuda.empty_cache()
    return reg, seq, u, host


def _slice_errors(out, ref, n):
    """max |out - ref| per 1/16 of the index range, relative to max |ref|."""
    scale = max(1.0, float(np.abs(ref).max()))
    parts = 16
    m = (1 << n) // parts
    return [float(np.abs(out[i * m:(i + 1) * m] - ref[i * m:(i + 1) * m]).max()) / scale for i in range(parts)]


@pytest.mark.parametrize("n,steps,cap", [(29, 8, 8), (30, 4, 4)])
def test_hpsi_whole_vector_vs_reference_matvec(rs, torch, n, steps, cap):
    from oracle import big

    name = "random29"
    reg, seq, u, psi = _mid_pulse_state(rs, torch, name, n, steps, cap, n_override=n)
    om, de = seq.step(steps)
    plan = rs.hamiltonian.context_for(n, u).pass_plan()
    if n == 29:
        assert [(p["a"], p["g"]) for p in plan] == [(12, 0), (3, 9), (4, 8)]
    else:
        assert [p["g"] for p in plan] == [0, 9, 9]
    s = rs.HamiltonianSlice.from_parameters(om, de, u)
    x = torch.from_numpy(psi).cuda()
    out = rs.apply_hamiltonian(s, x).cpu().numpy()
    del x
    torch.cuda.empty_cache()
    ham = big.HostHamiltonian(om, de, u)
    ref = ham.matvec(psi, np.empty_like(psi))
    errs = _slice_errors(out, ref, n)
    assert max(errs) <= 1e-12, {i: e for i, e in enumerate(errs) if e > 1e-12}
    # a spread-out state: every slice carries weight, so no slice is trivially zero
    m = (1 << n) // 16
    assert min(float(np.abs(psi[i * m:(i + 1) * m]).max()) for i in range(16)) > 0.0


@pytest.mark.parametrize("name,n,start,count,cap,max_vectors", [
    ("lattice27", 27, 30, 3, None, 40),    # configs[2]: 3 mid-pulse steps
    ("random29", 29, 8, 1, None, 17),      # configs[3]: 1 mid-pulse step (host basis <= 17 x 8.6 GB)
])
def test_lanczos_steps_vs_reference_algorithm(rs, torch, name, n, start, count, cap, max_vectors):
    from oracle import big
    from paper_2510_09813_b200.engine import SvEngine

    reg, seq, u, psi0 = _mid_pulse_state(rs, torch, name, n, start, cap or 20)
    masks = [1 << q for q in range(n)]

    # GPU: the fused Lanczos step (three-term recurrence, production kernels) from the same state
    eng = SvEngine(n, u, diag="fly", max_krylov_dim=100)
    try:
        eng.set_state(psi0)
        eng.set_observables(masks)
        gpu_iters, gpu_alpha0 = [], []
        for k in range(start, start + count):
            nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
            rep = eng.step(*seq.step(k), 10.0, 1e-10, 100, next_params=nxt, observe=True)
            assert rep.converged
            gpu_iters.append(rep.iterations)
            gpu_alpha0.append(rep.alpha0)
        gpu_occ = eng.observables()
        gpu_psi = eng.state().cpu().numpy()
    finally:
        eng.close()
        eng.slots = []
        del eng
        torch.cuda.empty_cache()

    # host: the reference's algorithm (full re-orthogonalisation) with the reference's matvec;
    # each step consumes its input (normalised in place as basis[0]) to bound host memory
    psi = psi0
    del psi0
    for i, k in enumerate(range(start, start + count)):
        om, de = seq.step(k)
        ham = big.HostHamiltonian(om, de, u)
        out, it, conv, res, alphas, _ = big.expm_multiply(ham, psi, 10.0, 1e-10, 100, max_vectors=max_vectors,
                                                          consume_input=True)
        assert conv
        assert abs(it - gpu_iters[i]) <= 1, (k, it, gpu_iters[i])
        assert abs(alphas[0] - gpu_alpha0[i]) <= 1e-8 * max(1.0, abs(alphas[0])), k   # Energy observable
        del ham
        psi = out
    fid = abs(big.vdot(psi, gpu_psi)) ** 2 / (big.norm(psi) ** 2 * big.norm(gpu_psi) ** 2)
    assert 1.0 - fid <= 1e-10
    p = np.abs(psi) ** 2
    total = p.sum()
    ref_occ = np.array([p.reshape(-1, 2, 1 << q)[:, 1, :].sum() / total for q in range(n)])
    assert np.abs(gpu_occ - ref_occ).max() <= 1e-8
    assert abs(math.sqrt(total) - 1.0) <= 1e-9
