"""Multi-process (world_size 2 and 4, gloo, CPU) checks of the top-qubit sharding host logic.

The shard-local arithmetic is a numpy stand-in built from the oracle (test infrastructure); the
code under test is paper_2510_09813_b200/sharding.py: effective detunings and offsets, partner
exchanges, all-reduced Lanczos scalars and observables. A sharded evolution must reproduce the
unsharded oracle evolution.
"""

import os
import socket

import numpy as np
import pytest

from oracle import sv_oracle as O


class NumpyLocalOps:
    def apply_local(self, om, de, u, x):
        return O.apply_hamiltonian(om, O.build_diagonal(de, u), x)

    def axpy(self, y, x, a):
        y += a * x

    def vdot(self, a, b):
        return complex(np.vdot(a, b))

    def copy(self, x):
        return np.array(x, copy=True)

    def scaled(self, x, a):
        return x * a

    def zeros_like(self, x):
        return np.zeros_like(x)

    def occupations_unnormalised(self, psi):
        n = int(np.log2(len(psi)))
        p = np.abs(psi) ** 2
        idx = np.arange(len(psi))
        return np.array([p[((idx >> q) & 1) == 1].sum() for q in range(n)]), float(p.sum())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, steps, outdir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_09813_b200.sharding import (ShardPlan, ShardedOperator, TorchComm, sharded_expm_multiply,
                                                 sharded_occupations)

    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 20, (n, 2))
    u = O.interaction_matrix(pos, 5.0e4)
    omegas = rng.uniform(0.5, 4.0, (steps, n))
    deltas = rng.uniform(-3.0, 3.0, (steps, n))
    plan = ShardPlan(n, world, rank)
    psi_full = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    psi_full /= np.linalg.norm(psi_full)
    psi = psi_full[plan.local_slice()].copy()
    ops, comm = NumpyLocalOps(), TorchComm(dist)
    for k in range(steps):
        op = ShardedOperator(plan, ops, comm, omegas[k], deltas[k], u)
        psi, it, conv, res = sharded_expm_multiply(op, psi, 10.0, 1e-12)
        assert conv
    occ = sharded_occupations(plan, ops, comm, psi)
    np.save(os.path.join(outdir, f"shard{rank}.npy"), psi)
    if rank == 0:
        np.save(os.path.join(outdir, "occ.npy"), occ)
        np.save(os.path.join(outdir, "inputs.npy"), {"u": u, "om": omegas, "de": deltas, "psi0": psi_full},
                allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_evolution_matches_oracle(tmp_path, world):
    import torch.multiprocessing as mp

    n, steps = 7, 3
    mp.spawn(_worker, args=(world, _free_port(), n, steps, str(tmp_path)), nprocs=world, join=True)
    shards = [np.load(tmp_path / f"shard{r}.npy") for r in range(world)]
    psi = np.concatenate(shards)
    inp = np.load(tmp_path / "inputs.npy", allow_pickle=True).item()
    ref = O.evolve_sv(inp["om"], inp["de"], 10, inp["u"], tolerance=1e-12, initial=inp["psi0"])
    assert np.linalg.norm(psi - ref["final_state"]) <= 1e-9
    occ = np.load(tmp_path / "occ.npy")
    assert np.abs(occ - O.occupations(ref["final_state"])).max() <= 1e-12


def test_effective_parameters_reproduce_the_diagonal():
    from paper_2510_09813_b200.sharding import ShardPlan

    rng = np.random.default_rng(1)
    n, world = 6, 4
    u = np.triu(rng.uniform(0, 2, (n, n)), 1)
    u = u + u.T
    de = rng.uniform(-2, 2, n)
    full = O.build_diagonal(de, u)
    for r in range(world):
        plan = ShardPlan(n, world, r)
        om, d_eff, u_loc, off, flips = plan.local_parameters(np.ones(n), de, u)
        local = O.build_diagonal(d_eff, u_loc) + off
        assert np.abs(local - full[plan.local_slice()]).max() <= 1e-12
        assert [f[2] for f in flips] == [r ^ 1, r ^ 2]


def test_plan_validation():
    from paper_2510_09813_b200.errors import ValidationError
    from paper_2510_09813_b200.sharding import ShardPlan

    with pytest.raises(ValidationError):
        ShardPlan(5, 3, 0)
    with pytest.raises(ValidationError):
        ShardPlan(2, 4, 0)
    p = ShardPlan(33, 8, 5)
    assert p.n_local == 30 and p.global_qubits == [30, 31, 32] and p.partner(31) == 7


def _comm_worker(rank, world, port, outdir):
    """FusedShardEngine's collective callback (the function the C driver calls through rsv_comm_fn),
    driven directly on host tensors over gloo: all-reduce in place, pairwise exchange into the buffer."""
    import ctypes

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_09813_b200 import _native as nat
    from paper_2510_09813_b200.sharding import FusedShardEngine

    eng = FusedShardEngine.__new__(FusedShardEngine)   # no GPU: only the callback is exercised
    eng.torch, eng.nat, eng.dist, eng.nccl = torch, nat, dist, False
    eng.device = torch.device("cpu")
    eng._reqs, eng._recv_host = [], None

    class _Slots:
        slots = [torch.full((8,), complex(rank, -rank), dtype=torch.complex128), torch.zeros(8, dtype=torch.complex128)]

    eng.eng = _Slots()
    eng.xbuf = torch.zeros(8, dtype=torch.complex128)
    vals = (ctypes.c_double * 3)(1.0 + rank, 10.0 * rank, -1.0)
    ok = [eng._comm(None, nat.RSV_COMM_ALLREDUCE, -1, -1, vals, 3)]
    peer = rank ^ 1
    ok.append(eng._comm(None, nat.RSV_COMM_EXCHANGE_START, 0, peer, None, 0))
    ok.append(eng._comm(None, nat.RSV_COMM_EXCHANGE_WAIT, 0, peer, None, 0))
    ok.append(eng._comm(None, 99, 0, 0, None, 0))
    np.save(os.path.join(outdir, f"c{rank}.npy"), {"ok": ok, "vals": list(vals), "x": eng.xbuf.numpy()},
            allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_fused_shard_comm_callback(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_comm_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        d = np.load(tmp_path / f"c{r}.npy", allow_pickle=True).item()
        assert d["ok"][:3] == [0, 0, 0] and d["ok"][3] != 0   # unknown op is reported, not ignored
        assert d["vals"] == [3.0, 10.0, -2.0]
        assert np.array_equal(d["x"], np.full(8, complex(r ^ 1, -(r ^ 1))))
