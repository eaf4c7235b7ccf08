"""Device-resident state-vector engine: one ``rsv_context`` plus its HBM workspace.

PyTorch is the plumbing here: it owns the device allocations (the Krylov slots)
and the CUDA stream; every byte of arithmetic runs in ``_rsv.so``.

HBM layout for N qubits (16 B per amplitude, 2^N amplitudes per vector):
  slots[0 .. K-1] Krylov basis s_0..s_{K-1} (s_0 is the state), unnormalised
  slots[K]        Lanczos iteration K-1's partial sums / residual (iteration j keeps its
                  partial sums u in slot j+1 and turns them into s_{j+1} in place; the
                  Krylov combination overwrites s_0 in place)
  dvec            optional 2^N float64 interaction diagonal (diag="vec" only)
K is min(max_krylov_dim, what fits in free HBM); steps that would need more
vectors are split exactly in time by the driver (rsv_capi.cu).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .errors import MemoryBudgetError, ValidationError

KMAX_NATIVE = 120         # rsv::kMaxKrylov
RESERVE_BYTES = 1 << 30   # headroom left to torch / the driver


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise nat.NativeError("no CUDA device: the state-vector hot path has no CPU fallback")
    return torch


def _cur_stream(torch, device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Context:
    """Thin owner of an ``rsv_context`` (no vectors bound): H.psi, observables, vector kernels."""

    def __init__(self, n_qubits: int, interaction_u, diag: str = "fly", device=None):
        torch = _torch()
        self.torch = torch
        self.lib = nat.load()
        self.n = int(n_qubits)
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.diag = diag
        mode = {"fly": nat.RSV_DIAG_FLY, "vec": nat.RSV_DIAG_VEC}.get(diag)
        if mode is None:
            raise ValidationError(f"diag must be 'fly' or 'vec', got {diag!r}")
        u = np.ascontiguousarray(interaction_u, dtype=np.float64)
        if u.shape != (self.n, self.n):
            raise ValidationError(f"interaction matrix shape {u.shape} does not match {self.n} qubits")
        self.u = u
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            nat.check(self.lib.rsv_create(self.n, nat.dptr(u), mode, _cur_stream(torch, self.device),
                                          ctypes.byref(ctx)), "rsv_create")
        self.ctx = ctx

    def sync_stream(self):
        nat.check(self.lib.rsv_set_stream(self.ctx, _cur_stream(self.torch, self.device)))

    def pass_plan(self):
        buf = (ctypes.c_int * 64)()
        nat.check(self.lib.rsv_pass_plan(self.ctx, buf, 64))
        n = buf[0]
        out = []
        for i in range(n):
            a, p, g, lo, fam, gm = (buf[1 + 6 * i + k] for k in range(6))
            d = dict(a=a, p=p, g=g, lo=bool(lo), family=("lo", "mid", "last", "iter2")[fam])
            if gm:
                d.update(family="chunk", chunk_bits=12 + gm, m_tile=dict(a=12 - gm, p=12, g=gm))
            out.append(d)
        return out

    def set_reorthogonalize(self, on: bool):
        """Full re-orthogonalisation of the Lanczos basis (reference krylov.py:103-104), opt-in."""
        nat.check(self.lib.rsv_set_reorthogonalize(self.ctx, 1 if on else 0), "rsv_set_reorthogonalize")

    def set_tail_regeneration(self, on: bool):
        """Beyond the resident basis: ring + regeneration (default) or exact split in time (off)."""
        nat.check(self.lib.rsv_set_tail_regeneration(self.ctx, 1 if on else 0), "rsv_set_tail_regeneration")

    def set_speculation(self, mode: int):
        """Speculative launch of Lanczos iteration j+1 before j is tested: -1 auto (N <= 24), 0 off, 1 on."""
        nat.check(self.lib.rsv_set_speculation(self.ctx, int(mode)), "rsv_set_speculation")

    def set_fusion(self, mode: int):
        """Two-pass Lanczos iterations ([lo, last] plans, 16..21 qubits) in one cooperative launch:
        -1 auto (on), 0 off, 1 on."""
        nat.check(self.lib.rsv_set_fusion(self.ctx, int(mode)), "rsv_set_fusion")

    def set_plan(self, chunk_group_bits: int = -1, chunk_lag: int = -1):
        """Pass-plan override (tests/tuning): -1 auto, 0 plain passes, 3..9 force the chunk pass."""
        nat.check(self.lib.rsv_set_plan(self.ctx, int(chunk_group_bits), int(chunk_lag)), "rsv_set_plan")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.rsv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def free_device_bytes(device) -> int:
    """HBM a new workspace can take: the driver's free memory plus the blocks torch's caching
    allocator holds that no tensor uses (an earlier engine's workspace: the allocator reuses them,
    or releases them and retries when a request does not fit)."""
    torch = _torch()
    free, _total = torch.cuda.mem_get_info(device)
    return int(free + torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device))


def slots_that_fit(n_qubits: int, max_krylov_dim: int, diag: str, device, budget_bytes=None,
                   vector_cap=None) -> int:
    torch = _torch()
    slot_bytes = 16 << n_qubits
    want = min(int(max_krylov_dim), KMAX_NATIVE) + 1
    if vector_cap is not None:
        want = min(want, int(vector_cap) + 1)
    free = free_device_bytes(device)
    extra = (8 << n_qubits) if diag == "vec" else 0
    avail = free - RESERVE_BYTES - extra
    if budget_bytes is not None:
        avail = min(avail, int(budget_bytes) - extra)
    return int(min(want, max(0, avail // slot_bytes)))


class SvEngine(Context):
    """State + Krylov workspace resident in HBM for one register."""

    def __init__(self, n_qubits: int, interaction_u, *, diag: str = "fly", max_krylov_dim: int = 100,
                 device=None, memory_budget_bytes=None, krylov_vectors_cap=None):
        super().__init__(n_qubits, interaction_u, diag=diag, device=device)
        torch = self.torch
        nslots = slots_that_fit(self.n, max_krylov_dim, diag, self.device, memory_budget_bytes,
                                krylov_vectors_cap)
        if nslots < 3:
            need = (16 << self.n) * 3
            raise MemoryBudgetError(
                f"state-vector workspace for N={self.n} needs at least {need:.3e} bytes of HBM "
                "(state + two Lanczos vectors)", required_bytes=need, budget_bytes=memory_budget_bytes)
        with torch.cuda.device(self.device):
            self.slots = [torch.empty(1 << self.n, dtype=torch.complex128, device=self.device)
                          for _ in range(nslots)]
            ptrs = (ctypes.c_void_p * nslots)(*[t.data_ptr() for t in self.slots])
            nat.check(self.lib.rsv_bind_slots(self.ctx, ptrs, nslots), "rsv_bind_slots")
            self.dvec = None
            if diag == "vec":
                self.dvec = torch.empty(1 << self.n, dtype=torch.float64, device=self.device)
                self.sync_stream()
                nat.check(self.lib.rsv_bind_diag_vector(self.ctx, ctypes.c_void_p(self.dvec.data_ptr()), 1))
        self.krylov_cap = nslots - 1
        self.masks = np.zeros(0, dtype=np.uint64)
        self.set_basis_state(0)

    # -- state ---------------------------------------------------------------
    def state(self):
        """The resident state (a view into the workspace; the next step reuses it)."""
        idx = ctypes.c_int()
        nat.check(self.lib.rsv_state_slot(self.ctx, ctypes.byref(idx)))
        return self.slots[idx.value]

    def set_basis_state(self, bits: int):
        psi = self.state()
        psi.zero_()
        psi[int(bits)] = 1.0
        nat.check(self.lib.rsv_state_modified(self.ctx))

    def set_state(self, psi):
        torch = self.torch
        dst = self.state()
        if isinstance(psi, np.ndarray):
            src = torch.from_numpy(np.ascontiguousarray(psi, dtype=np.complex128))
            if src.shape != dst.shape:
                raise ValidationError(f"initial state has shape {tuple(src.shape)}, expected ({dst.numel()},)")
            dst.copy_(src)
        else:
            if tuple(psi.shape) != tuple(dst.shape):
                raise ValidationError(f"initial state has shape {tuple(psi.shape)}, expected ({dst.numel()},)")
            dst.copy_(psi.to(torch.complex128))
        nat.check(self.lib.rsv_state_modified(self.ctx))

    # -- observables ---------------------------------------------------------
    def set_observables(self, masks):
        self.masks = np.ascontiguousarray(np.asarray(masks, dtype=np.uint64))
        nat.check(self.lib.rsv_set_observables(
            self.ctx, self.masks.ctypes.data_as(nat.c_u64_p), int(self.masks.size)))

    def observables(self) -> np.ndarray:
        out = np.zeros(max(1, self.masks.size))
        nat.check(self.lib.rsv_get_observables(self.ctx, nat.dptr(out)))
        return out[: self.masks.size]

    def measure(self):
        out = np.zeros(max(1, self.masks.size))
        nsq = ctypes.c_double()
        self.sync_stream()
        nat.check(self.lib.rsv_measure(self.ctx, nat.dptr(out), ctypes.byref(nsq)))
        return out[: self.masks.size], nsq.value

    # -- hot path --------------------------------------------------------------
    def step(self, omegas, deltas, dt_ns: float, tolerance: float, max_krylov_dim: int,
             norm_epsilon: float = 1e-14, next_params=None, observe: bool = False):
        om = np.ascontiguousarray(omegas, dtype=np.float64)
        de = np.ascontiguousarray(deltas, dtype=np.float64)
        if om.shape != (self.n,) or de.shape != (self.n,):
            raise ValidationError(f"step parameters must have shape ({self.n},)")
        nom = nde = None
        if next_params is not None:
            nom = np.ascontiguousarray(next_params[0], dtype=np.float64)
            nde = np.ascontiguousarray(next_params[1], dtype=np.float64)
        rep = nat.KrylovReportC()
        self.sync_stream()
        nat.check(self.lib.rsv_expm_step(
            self.ctx, nat.dptr(om), nat.dptr(de), float(dt_ns), float(tolerance), int(max_krylov_dim),
            float(norm_epsilon), nat.dptr(nom) if nom is not None else None,
            nat.dptr(nde) if nde is not None else None, 1 if observe else 0, ctypes.byref(rep)),
            "rsv_expm_step")
        return rep

    # -- profiling -----------------------------------------------------------------
    def set_profiling(self, on, every: int = 1):
        """Kernel timing by CUDA events (profile()); ``every``: time one launch in that many per
        kernel family (the per-launch event pair costs host time on small registers)."""
        nat.check(self.lib.rsv_set_profiling(self.ctx, max(1, int(every)) if on else 0))
        nat.check(self.lib.rsv_reset_profile(self.ctx))

    def profile(self):
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_longlong * 4)()
        nat.check(self.lib.rsv_get_profile(self.ctx, ms, cnt))
        p0 = self.pass_plan()[0]
        first = p0["family"] if p0["family"] in ("chunk", "iter2") else ("lo" if p0["lo"] else "first")
        names = (first, "mid", "last", "combine")
        return {names[i]: {"ms": ms[i], "launches": cnt[i]} for i in range(4)}
