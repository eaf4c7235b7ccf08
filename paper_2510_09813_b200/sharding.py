"""State sharding by the top log2(P) qubits across P processes (one GPU each).

North-star row (e): an N-qubit state is split into P = 2^k contiguous shards of 2^(N-k)
amplitudes; rank r holds the indices whose top k bits equal r. Then

* every flip on a local qubit (i < N-k) and every diagonal term are shard-local: the local
  passes run unchanged with *effective* detunings
      delta_eff_i = delta_i - sum_{g global, bit_g(r)=1} U_ig
  and a constant per-rank energy offset
      E_r = -sum_{g set} delta_g + sum_{g<g' set} U_gg';
* a flip on a global qubit g is the elementwise exchange
      y_r += (Omega_g / 2) * psi_{r ^ 2^(g-N+k)}
  with the partner rank (NCCL send/recv or P2P loads over NVLink);
* the Lanczos scalars (alpha, beta, norms) and observables are all-reduced.

This module holds that host-side logic. It is backend-agnostic: a ``LocalOps`` object supplies
the shard-local arithmetic (the rsv C ABI on a GPU; the CPU tests plug a numpy restatement) and a
``Comm`` object the exchange/all-reduce (torch.distributed: NCCL on GPUs, gloo in the CPU tests).
The reference algorithm of rydsim/krylov.py:67-125 (with its full re-orthogonalisation) runs on
top, so a sharded run is checked against the unsharded oracle.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import MemoryBudgetError, ValidationError

NS_TO_US = 1e-3
_BREAKDOWN_RTOL = 1e-14


@dataclass(frozen=True)
class ShardPlan:
    n_qubits: int
    world_size: int
    rank: int

    def __post_init__(self):
        p = self.world_size
        if p < 1 or p & (p - 1):
            raise ValidationError(f"world size {p} is not a power of two")
        if not 0 <= self.rank < p:
            raise ValidationError(f"rank {self.rank} outside [0, {p})")
        if self.n_global >= self.n_qubits:
            raise ValidationError(f"{p} shards need more than {self.n_global} qubits")

    @property
    def n_global(self) -> int:
        return int(math.log2(self.world_size))

    @property
    def n_local(self) -> int:
        return self.n_qubits - self.n_global

    @property
    def global_qubits(self):
        return list(range(self.n_local, self.n_qubits))

    def global_bit(self, q: int) -> int:
        return (self.rank >> (q - self.n_local)) & 1

    def partner(self, q: int) -> int:
        """Rank holding the amplitudes with qubit q (global) flipped."""
        return self.rank ^ (1 << (q - self.n_local))

    def local_slice(self):
        size = 1 << self.n_local
        return slice(self.rank * size, (self.rank + 1) * size)

    def local_parameters(self, omegas, deltas, u):
        """(local omegas, effective local deltas, local U, energy offset, global flips).

        global flips: list of (qubit, Omega_q / 2, partner rank) for nonzero drives.
        """
        omegas = np.asarray(omegas, dtype=float)
        deltas = np.asarray(deltas, dtype=float)
        u = np.asarray(u, dtype=float)
        nl = self.n_local
        set_g = [g for g in self.global_qubits if self.global_bit(g)]
        d_eff = deltas[:nl].copy()
        for g in set_g:
            d_eff -= u[:nl, g]
        offset = -sum(deltas[g] for g in set_g)
        for a_i, g in enumerate(set_g):
            for h in set_g[a_i + 1:]:
                offset += u[g, h]
        flips = [(g, 0.5 * omegas[g], self.partner(g)) for g in self.global_qubits if omegas[g] != 0.0]
        return omegas[:nl].copy(), d_eff, u[:nl, :nl].copy(), float(offset), flips


class ShardedOperator:
    """y = H psi for a sharded psi: local passes + offset + partner exchanges."""

    def __init__(self, plan: ShardPlan, local_ops, comm, omegas, deltas, u):
        self.plan = plan
        self.ops = local_ops
        self.comm = comm
        self.om, self.de, self.u, self.offset, self.flips = plan.local_parameters(omegas, deltas, u)

    def __call__(self, x):
        y = self.ops.apply_local(self.om, self.de, self.u, x)
        if self.offset != 0.0:
            self.ops.axpy(y, x, self.offset)
        for _q, coef, partner in self.flips:
            peer = self.comm.exchange(x, partner)
            self.ops.axpy(y, peer, coef)
        return y


def tridiag_exp_e1(alphas, betas, tau):
    """exp(-1j tau T) e1 (krylov.py:54) by the step driver's routine (rsv_tridiag_exp_e1)."""
    return nat.tridiag_exp_e1(alphas, betas, tau)


def sharded_expm_multiply(op: ShardedOperator, psi, dt_ns, tolerance=1e-10, max_krylov_dim=100,
                          norm_epsilon=1e-14):
    """krylov.py:67-125 over shards: every inner product is an all-reduce."""
    ops, comm = op.ops, op.comm

    def dot(a, b):
        return comm.allreduce_complex(ops.vdot(a, b))

    norm_in = math.sqrt(max(0.0, dot(psi, psi).real))
    if norm_in <= norm_epsilon:
        return ops.copy(psi), 0, True, 0.0
    if dt_ns == 0.0:
        return ops.copy(psi), 1, True, 0.0
    tau = dt_ns * NS_TO_US
    basis = [ops.scaled(psi, 1.0 / norm_in)]
    alphas, betas = [], []
    converged = False
    residual = math.inf
    while True:
        w = op(basis[-1])
        a = dot(basis[-1], w).real
        alphas.append(a)
        ops.axpy(w, basis[-1], -a)
        if betas:
            ops.axpy(w, basis[-2], -betas[-1])
        for v in basis:
            ops.axpy(w, v, -dot(v, w))
        b = math.sqrt(max(0.0, dot(w, w).real))
        y = tridiag_exp_e1(alphas, betas, tau)
        residual = b * abs(y[-1])
        scale = max(1.0, max(abs(x) for x in alphas), max(betas, default=0.0))
        if residual <= tolerance or b <= _BREAKDOWN_RTOL * scale:
            converged = True
            break
        if len(alphas) >= max_krylov_dim:
            break
        betas.append(b)
        basis.append(ops.scaled(w, 1.0 / b))
    out = ops.zeros_like(psi)
    for coef, v in zip(y, basis):
        ops.axpy(out, v, complex(coef) * norm_in)
    return out, len(alphas), converged, float(residual)


def sharded_occupations(plan: ShardPlan, local_ops, comm, psi):
    """<n_q> for all N qubits: local bits reduce on the shard, global bits are rank constants."""
    local_occ, local_norm = local_ops.occupations_unnormalised(psi)
    tot = comm.allreduce_real(np.concatenate([local_occ, [local_norm]]))
    occ_local = tot[:-1] / tot[-1]
    glob = np.array([plan.global_bit(g) * local_norm for g in plan.global_qubits])
    glob = comm.allreduce_real(glob) / tot[-1]
    return np.concatenate([occ_local, glob])


class TorchComm:
    """Exchange / all-reduce over torch.distributed (NCCL on GPUs, gloo in CPU tests)."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.device = device

    def exchange(self, x, partner):
        import torch

        send = torch.as_tensor(x)
        staged = send.is_cuda and self.dist.get_backend() == "gloo"
        if staged:   # gloo moves host tensors only
            send = send.cpu()
        recv = torch.empty_like(send)
        rank = self.dist.get_rank()
        # deadlock-free pairwise exchange: the lower rank sends first
        if rank < partner:
            self.dist.send(send, partner)
            self.dist.recv(recv, partner)
        else:
            self.dist.recv(recv, partner)
            self.dist.send(send, partner)
        if staged:
            return recv.to(x.device)
        return recv if not isinstance(x, np.ndarray) else recv.numpy()

    def allreduce_real(self, arr):
        import torch

        t = torch.as_tensor(np.asarray(arr, dtype=np.float64).copy())
        if self.device is not None:
            t = t.to(self.device)
        self.dist.all_reduce(t)
        return t.cpu().numpy()

    def allreduce_complex(self, z):
        r = self.allreduce_real([z.real, z.imag])
        return complex(r[0], r[1])


class CudaLocalOps:
    """Shard-local arithmetic on the GPU through the rsv C ABI (no CPU fallback).

    The local operator is the n_local-qubit Rydberg Hamiltonian with the effective detunings
    of the shard (``ShardPlan.local_parameters``) applied by the bit-group pass kernels; the
    vector algebra uses the rsv vector kernels.
    """

    def __init__(self, n_local: int, u_local, device=None):
        import ctypes

        from .engine import Context

        self.ctypes = ctypes
        self.ctx = Context(n_local, u_local, diag="fly", device=device)
        self.lib = self.ctx.lib
        self.torch = self.ctx.torch
        self.n = n_local

    def _c(self):
        self.ctx.sync_stream()
        return self.ctx.ctx

    def apply_local(self, om, de, u, x):
        from . import _native as nat

        om = np.ascontiguousarray(om, dtype=np.float64)
        de = np.ascontiguousarray(de, dtype=np.float64)
        y = self.torch.empty_like(x)
        nat.check(self.lib.rsv_apply_hamiltonian(self._c(), nat.dptr(om), nat.dptr(de), x.data_ptr(), y.data_ptr()))
        return y

    def axpy(self, y, x, a):
        from . import _native as nat

        a = complex(a)
        nat.check(self.lib.rsv_axpy(self._c(), y.data_ptr(), x.data_ptr(), a.real, a.imag, x.numel()))

    def vdot(self, a, b):
        from . import _native as nat

        out = (self.ctypes.c_double * 2)()
        nat.check(self.lib.rsv_zdotc(self._c(), a.data_ptr(), b.data_ptr(), a.numel(), out))
        return complex(out[0], out[1])

    def copy(self, x):
        return x.clone()

    def scaled(self, x, a):
        from . import _native as nat

        y = self.torch.empty_like(x)
        a = complex(a)
        nat.check(self.lib.rsv_scale(self._c(), y.data_ptr(), x.data_ptr(), a.real, a.imag, x.numel()))
        return y

    def zeros_like(self, x):
        return self.torch.zeros_like(x)

    def occupations_unnormalised(self, psi):
        from . import _native as nat

        masks = np.ascontiguousarray([1 << q for q in range(self.n)], dtype=np.uint64)
        out = np.zeros(self.n)
        nsq = self.ctypes.c_double()
        nat.check(self.lib.rsv_observe(self._c(), psi.data_ptr(), masks.ctypes.data_as(nat.c_u64_p), self.n,
                                       nat.dptr(out), self.ctypes.byref(nsq)))
        return out * nsq.value, float(nsq.value)


def evolve_sv_sharded(seq, reg, dist, tolerance=1e-10, max_krylov_dim=100, initial_local=None, device=None):
    """Sharded exact evolution (row e): every rank holds 2^(N - log2 P) amplitudes on its GPU.

    Partner exchanges go through torch.distributed (NCCL send/recv on GPUs; the gloo test path
    stages through host memory). Returns (local final state, per-step iterations, occupations).
    """
    import torch

    from .hamiltonian import interaction_matrix

    n = reg.qubit_count
    plan = ShardPlan(n, dist.get_world_size(), dist.get_rank())
    u = interaction_matrix(reg)
    ops = CudaLocalOps(plan.n_local, u[:plan.n_local, :plan.n_local], device=device)
    comm = TorchComm(dist, device=ops.ctx.device if dist.get_backend() == "nccl" else None)
    if initial_local is None:
        psi = torch.zeros(1 << plan.n_local, dtype=torch.complex128, device=ops.ctx.device)
        if plan.rank == 0:
            psi[0] = 1.0
    else:
        psi = initial_local.to(ops.ctx.device, torch.complex128).clone()
    iters = []
    for k in range(seq.step_count):
        om, de = seq.step(k)
        op = ShardedOperator(plan, ops, comm, om, de, u)
        psi, it, conv, res = sharded_expm_multiply(op, psi, float(seq.dt_ns), tolerance, max_krylov_dim)
        if not conv:
            from .errors import SolverError

            raise SolverError(f"Krylov did not converge at step {k} (residual {res:.3e})", step=k, residual=res)
        iters.append(it)
    occ = sharded_occupations(plan, ops, comm, psi)
    return psi, iters, occ


class FusedShardEngine:
    """One shard of a sharded exact evolution on the fused Lanczos driver (rsv_expm_step).

    The local qubits run the same bit-group pass kernels as a single GPU (effective detunings and
    the shard's constant energy folded into the diagonal tables); the driver calls back into this
    object for the collectives (include/rsv.h, rsv_comm_fn): all-reduces of the Lanczos scalars
    (alpha partial, ||w||^2, <w|A_last|w>, ||psi||^2, observables) and, per global qubit with a
    nonzero drive, the exchange of s_j with the partner shard -- the first one started before the
    local passes so that it overlaps them (NCCL on its own stream); its flip and share of alpha
    are applied by the global_flip kernel before the last pass.
    """

    def __init__(self, n_qubits: int, u, dist, *, device=None, max_krylov_dim: int = 100,
                 memory_budget_bytes=None, krylov_vectors_cap=None, initial_local=None, peer_memory=False,
                 device_scalars=True):
        import ctypes

        import torch

        from . import _native as nat
        from .engine import SvEngine

        self.torch = torch
        self.nat = nat
        self.dist = dist
        self.plan = ShardPlan(n_qubits, dist.get_world_size(), dist.get_rank())
        self.u = np.asarray(u, dtype=float)
        nl = self.plan.n_local
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        # bring up the communicator before the workspace takes the GPU's memory (NCCL allocates
        # its buffers lazily at the first collective / the first pairwise exchange), and leave it
        # a few GB: the Krylov slots otherwise take all of HBM
        dist.barrier()
        if memory_budget_bytes is None:
            from .engine import free_device_bytes

            memory_budget_bytes = max(0, free_device_bytes(dev) - (4 << 30))
        # every rank must stop its Lanczos loop (and split a step) at the same Krylov cap, or the
        # shards would enter different collectives: agree on the smallest slot count that fits
        from .engine import slots_that_fit

        local = slots_that_fit(nl, max_krylov_dim, "fly", dev, memory_budget_bytes, krylov_vectors_cap)
        agreed = torch.tensor([float(local)], dtype=torch.float64,
                              device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(agreed, op=dist.ReduceOp.MIN)
        nslots = int(agreed.item())
        self.eng = SvEngine(nl, self.u[:nl, :nl], diag="fly", max_krylov_dim=max_krylov_dim, device=dev,
                            memory_budget_bytes=memory_budget_bytes, krylov_vectors_cap=max(0, nslots - 1))
        if len(self.eng.slots) != nslots:   # pragma: no cover - the budget shrank between the two queries
            raise MemoryBudgetError(f"rank {dist.get_rank()}: {len(self.eng.slots)} Krylov slots, the ranks agreed "
                                    f"on {nslots}")
        self.nccl = dist.get_backend() == "nccl"
        self._reqs = []
        self._recv_host = None
        self.peer_memory = False
        self._peer_tensors = []
        plan = self.eng.pass_plan()
        if peer_memory and len(plan) > 1 and plan[0]["family"] != "chunk":   # else the exchange is used
            self.peer_memory = self._map_peers()
        # exchange mode needs a buffer for the partner's copy: a small one, or the last Krylov slot
        # when the shard is large (all of HBM went to the slots)
        self.xbuf = None
        if not self.peer_memory:
            if nl <= 20 or len(self.eng.slots) < 4:
                self.xbuf = torch.empty(1 << nl, dtype=torch.complex128, device=dev)
            else:
                self.xbuf = self.eng.slots.pop()
                ptrs = (ctypes.c_void_p * len(self.eng.slots))(*[t.data_ptr() for t in self.eng.slots])
                nat.check(self.eng.lib.rsv_bind_slots(self.eng.ctx, ptrs, len(self.eng.slots)), "rsv_bind_slots")
                self.eng.krylov_cap -= 1
        self._cb = nat.COMM_FN(self._comm)   # keep the ctypes thunk alive
        nat.check(self.eng.lib.rsv_set_shard(self.eng.ctx, self._cb, None,
                                             self.xbuf.data_ptr() if self.xbuf is not None else None),
                  "rsv_set_shard")
        # on-stream all-reduces of the per-iteration Lanczos scalars (RSV_COMM_ALLREDUCE_DEVICE): the
        # peer-memory iteration then has no host round trip (device_scalars=False: host path)
        self.red = torch.zeros(8, dtype=torch.float64, device=dev)
        self.device_scalars = bool(device_scalars)
        if self.device_scalars:
            nat.check(self.eng.lib.rsv_set_shard_scratch(self.eng.ctx, ctypes.c_void_p(self.red.data_ptr()), 8),
                      "rsv_set_shard_scratch")
        self.eng.set_observables([1 << q for q in range(nl)])
        psi = self.eng.state()
        if initial_local is not None:   # this shard's amplitudes (host or device tensor)
            if tuple(initial_local.shape) != (1 << nl,):
                raise ValidationError(f"initial shard has shape {tuple(initial_local.shape)}, expected ({1 << nl},)")
            psi.copy_(initial_local, non_blocking=True)
        else:
            psi.zero_()
            if self.plan.rank == 0:
                psi[0] = 1.0   # |0...0>: every global bit 0 lives on rank 0
        nat.check(self.eng.lib.rsv_state_modified(self.eng.ctx))

    def _map_peers(self) -> bool:
        """Peer-memory mode: map every partner shard's Krylov slots into this process (CUDA IPC;
        on an NVLink box the mapping is a peer mapping, so the first pass reads them with P2P
        loads). All ranks agree on the outcome; on any failure they stay in exchange mode."""
        import ctypes

        from torch.multiprocessing.reductions import reduce_tensor

        torch, dist, nat = self.torch, self.dist, self.nat
        ok = 1.0
        try:
            mine = [reduce_tensor(t) for t in self.eng.slots]
            everyone = [None] * dist.get_world_size()
            dist.all_gather_object(everyone, mine)
            table = []
            for g in self.plan.global_qubits:
                peer = self.plan.partner(g)
                if len(everyone[peer]) != len(self.eng.slots):
                    raise RuntimeError(f"partner rank {peer} has {len(everyone[peer])} slots, this rank "
                                       f"{len(self.eng.slots)}")
                tensors = [fn(*args) for fn, args in everyone[peer]]
                self._peer_tensors.append(tensors)
                table.extend(t.data_ptr() for t in tensors)
            with torch.cuda.device(self.device):   # kernels on this GPU read the partners' memory
                for p in table[:: len(self.eng.slots)]:
                    nat.check(self.eng.lib.rsv_enable_peer_access(p), "rsv_enable_peer_access")
        except Exception:   # pragma: no cover - platform without CUDA IPC / P2P
            ok = 0.0
        flag = torch.tensor([ok], dtype=torch.float64, device=self.device if self.nccl else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() < 1.0:
            self._peer_tensors = []
            return False
        ng, ns = len(self.plan.global_qubits), len(self.eng.slots)
        arr = (ctypes.c_void_p * (ng * ns))(*table)
        nat.check(self.eng.lib.rsv_set_shard_peers(self.eng.ctx, ng, arr, ns), "rsv_set_shard_peers")
        return True

    # -- collectives requested by the C driver --------------------------------------
    def _comm(self, _user, op, slot, peer, host, count):
        try:
            torch, dist, nat = self.torch, self.dist, self.nat
            if op == nat.RSV_COMM_ALLREDUCE_DEVICE:
                # `host` points into self.red (device): in-place sum on the current stream (the
                # context's); NCCL orders it with the stream's kernels, nothing waits on the host
                dist.all_reduce(self.red[:count])
            elif op == nat.RSV_COMM_ALLREDUCE:
                arr = np.ctypeslib.as_array(host, shape=(count,))
                t = torch.from_numpy(arr.copy())
                if self.nccl:
                    t = t.to(self.device)
                dist.all_reduce(t)
                arr[:] = t.cpu().numpy()
            elif op == nat.RSV_COMM_EXCHANGE_START:
                send = self.eng.slots[slot]
                if self.nccl:   # NCCL P2P on its own stream: overlaps the local passes
                    ops = [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, self.xbuf, peer)]
                else:           # gloo moves host tensors (CPU tests / one-GPU test boxes)
                    self._send_host = send.cpu()
                    self._recv_host = torch.empty_like(self._send_host)
                    ops = [dist.P2POp(dist.isend, self._send_host, peer),
                           dist.P2POp(dist.irecv, self._recv_host, peer)]
                self._reqs = dist.batch_isend_irecv(ops)
            elif op == nat.RSV_COMM_EXCHANGE_WAIT:
                for r in self._reqs:
                    r.wait()
                self._reqs = []
                if not self.nccl:
                    self.xbuf.copy_(self._recv_host)
                if self.xbuf.is_cuda:
                    torch.cuda.current_stream(self.device).synchronize()
            else:
                return 2
            return 0
        except Exception:   # pragma: no cover - reported through the C error path
            import traceback

            traceback.print_exc()
            return 1

    # -- one exact step ------------------------------------------------------------
    def _local(self, omegas, deltas):
        om_l, de_eff, _u, offset, _flips = self.plan.local_parameters(omegas, deltas, self.u)
        coef = np.array([0.5 * float(omegas[g]) for g in self.plan.global_qubits], dtype=np.float64)
        peer = np.array([self.plan.partner(g) for g in self.plan.global_qubits], dtype=np.int32)
        return om_l, de_eff, offset, coef, peer

    def step(self, omegas, deltas, dt_ns, tolerance=1e-10, max_krylov_dim=100, next_params=None,
             observe=False, norm_epsilon=1e-14):
        import ctypes

        nat = self.nat
        om_l, de_eff, offset, coef, peer = self._local(omegas, deltas)
        nxt = None
        next_offset = offset
        if next_params is not None:
            n_om, n_de, next_offset, _c, _p = self._local(*next_params)
            nxt = (n_om, n_de)
        self.eng.sync_stream()
        nat.check(self.eng.lib.rsv_set_shard_step(
            self.eng.ctx, float(offset), float(next_offset), len(coef), nat.dptr(coef),
            peer.ctypes.data_as(ctypes.POINTER(ctypes.c_int))), "rsv_set_shard_step")
        return self.eng.step(om_l, de_eff, dt_ns, tolerance, max_krylov_dim, norm_epsilon, next_params=nxt,
                             observe=observe)

    def occupations(self):
        """<n_q> for all N qubits after an observed step: local qubits from the all-reduced mask sums,
        global qubits from the shards' norms (rank bits)."""
        import ctypes

        occ_local = self.eng.observables()
        loc = ctypes.c_double()
        self.nat.check(self.eng.lib.rsv_shard_local_norm_sq(self.eng.ctx, ctypes.byref(loc)))
        vals = [self.plan.global_bit(g) * loc.value for g in self.plan.global_qubits] + [loc.value]
        tot = TorchComm(self.dist, self.device if self.nccl else None).allreduce_real(vals)
        return np.concatenate([occ_local, tot[:-1] / tot[-1]])

    def state(self):
        return self.eng.state()

    def peer_stats(self):
        """Peer-memory passes launched so far: {"tma": partner tiles by TMA into the shared-memory
        ring, "loads": per-thread P2P loads}."""
        out = (ctypes.c_longlong * 2)()
        self.nat.check(self.eng.lib.rsv_shard_peer_stats(self.eng.ctx, out))
        return {"tma": int(out[0]), "loads": int(out[1])}

    def close(self):
        self.nat.check(self.eng.lib.rsv_set_shard_peers(self.eng.ctx, 0, None, 0))
        self.nat.check(self.eng.lib.rsv_set_shard(self.eng.ctx, self.nat.COMM_FN(), None, None))
        self.dist.barrier()   # partners may still read this shard's slots until everyone is done
        self._peer_tensors = []
        if self.peer_memory:
            import gc

            gc.collect()
            self.dist.barrier()           # every rank has dropped its mappings of the others' slots
            self.torch.cuda.ipc_collect()  # so the exported blocks can really be freed
        self.eng.close()


def evolve_sv_sharded_fused(seq, reg, dist, tolerance=1e-10, max_krylov_dim=100, device=None,
                            krylov_vectors_cap=None, initial_local=None, peer_memory=False, info=None):
    """Sharded exact evolution on the fused kernels (row e): returns (local final state, per-step
    Krylov reports, occupations of all N qubits after the last step). ``initial_local``: this rank's
    2^(N - log2 P) amplitudes (default |0...0>). ``peer_memory``: read the partner shards through
    CUDA IPC mappings instead of exchanging copies (falls back to the exchange if unavailable;
    ``info["peer_memory"]`` tells which ran)."""
    from .errors import SolverError
    from .hamiltonian import interaction_matrix

    eng = FusedShardEngine(reg.qubit_count, interaction_matrix(reg), dist, device=device,
                           max_krylov_dim=max_krylov_dim, krylov_vectors_cap=krylov_vectors_cap,
                           initial_local=initial_local, peer_memory=peer_memory)
    if info is not None:   # which global-flip mode actually ran
        info["peer_memory"] = eng.peer_memory
    reps = []
    for k in range(seq.step_count):
        nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
        rep = eng.step(*seq.step(k), float(seq.dt_ns), tolerance, max_krylov_dim, next_params=nxt,
                       observe=(k + 1 == seq.step_count))
        if not rep.converged:
            raise SolverError(f"Krylov did not converge at step {k} (residual {rep.residual:.3e})", step=k,
                              residual=rep.residual)
        reps.append(rep)
    occ = eng.occupations()
    psi = eng.state().clone()
    if info is not None:   # peer-memory passes: partner tiles by TMA ring / per-thread P2P loads
        info["peer_passes"] = eng.peer_stats()
    eng.close()
    return psi, reps, occ
