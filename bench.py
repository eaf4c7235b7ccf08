#!/usr/bin/env python
"""Benchmark of the B200 state-vector hot path (BASELINE.json configs[3]: N=29 random 2D register,
per-atom detuning map, noiseless 1 us Rydberg pulse, dt = 10 ns -> 100 Krylov time steps).

A bench *step* is one exact time step psi <- exp(-i dt H_k) psi (one rsv_expm_step: the fused
Lanczos H.psi passes + Krylov combination + occupation reduction, and the host read of that
step's occupations). Default: W=3 warm-up steps then K=97 timed steps = the whole 1 us pulse.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--qubits 29] [--diag fly|vec]
                  [--workload random29|lattice27|lattice20|ring10] [--plan-gm G] [--total-qubits 33]

value = H.psi products per second (whole job); ms_per_step; s_per_us_pulse; effective HBM
GB/s (32 B per amplitude per H.psi: read psi, write H psi); roofline of the dominant kernel;
e2e through the public API (evolve_sv) with host initial/final state; CPU baseline (C port of
the reference's numba matvec, OpenMP on the host cores, bounded sample). Multi-GPU (torchrun, P GPUs):
one register of N = n + log2(P) qubits sharded by its top qubits (weak scaling; run_sharded; the
partner shards are read with P2P loads unless --no-peer-memory), max over ranks; --total-qubits
fixes N (strong scaling, BASELINE configs[4]); --replicas runs P independent single-GPU copies.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = None
try:
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        BASELINE_METRIC = json.load(fh)["metric"]
except Exception:  # pragma: no cover
    BASELINE_METRIC = "H.psi/sec and effective HBM GB/s at N=29 (1 GPU)/N=33 (8 GPU); s per 1 us pulse"


WORKLOAD_TEXT = {   # BASELINE.json configs
    "random29": ("random 2D register (mean spacing 7 um, min 6 um, C6 = 2pi*862690), per-atom detuning map "
                 "0.6..1, Blackman Omega peak 3pi rad/us, delta -6..6 rad/us, 1 us pulse (configs[3])"),
    "lattice27": ("3x9 square lattice, 6.5 um spacing, global Blackman pulse Omega peak 3pi rad/us, delta -6..6 "
                  "rad/us, 1 us (configs[2]: the paper's A100 40 GB limit)"),
    "lattice20": "4x5 square lattice, 5.6 um spacing, adiabatic delta sweep -6..6 rad/us over 3 us (configs[1])",
    "ring10": "ring register, constant Omega = 2pi rad/us, delta = 0, 1 us (configs[0])",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU baseline (oracle C port)
def cpu_baseline(n, seconds=12.0, chunk_log2=None, steps=None, warmup=1):
    """Time the C restatement of the reference's matvec (rydsim/_kernels.py:14) on the host cores.

    Bounded sample: each timed unit computes H.psi on a contiguous 1/2^k slice of the output
    (each element still reads all N partners across the full 2^n state). Returns H.psi/s.
    """
    import ctypes

    import psutil

    from oracle import build as obuild

    lib = obuild.load()
    # every host core this process may run on (torchrun sets OMP_NUM_THREADS=1 in each rank)
    lib.svref_set_threads(len(os.sched_getaffinity(0)))
    dp = ctypes.POINTER(ctypes.c_double)
    avail = psutil.virtual_memory().available
    n_used = n
    while n_used > 16 and (16 + 16 + 8) * (2 ** n_used) > 0.6 * avail:
        n_used -= 1
    dim = 2 ** n_used
    psi = np.empty(2 * dim)
    out = np.empty(2 * dim)
    diag = np.empty(dim)
    lib.svref_fill(2 * dim, psi.ctypes.data_as(dp), 1234)
    from paper_2510_09813_b200 import interaction_matrix, workloads

    reg, seq = workloads.config("random29", n_override=n_used)
    u = np.ascontiguousarray(interaction_matrix(reg))
    om, de = seq.step(50)
    lib.svref_build_diagonal(n_used, np.ascontiguousarray(de).ctypes.data_as(dp), u.ctypes.data_as(dp),
                             diag.ctypes.data_as(dp))
    h = np.ascontiguousarray(0.5 * om)
    if chunk_log2 is None:
        chunk_log2 = max(0, n_used - 24)
    chunk = dim >> chunk_log2
    nchunks = 1 << chunk_log2

    def run(i):
        b0 = (i % nchunks) * chunk
        lib.svref_matvec_range(n_used, psi.ctypes.data_as(dp), diag.ctypes.data_as(dp), h.ctypes.data_as(dp),
                               out.ctypes.data_as(dp), b0, b0 + chunk)

    for i in range(warmup):
        run(i)
    t0 = time.perf_counter()
    done = 0
    while True:
        run(done)
        done += 1
        el = time.perf_counter() - t0
        if (steps is not None and done >= steps) or (steps is None and el >= seconds):
            break
    el = time.perf_counter() - t0
    hpsi = done / nchunks
    # scale to the requested N if the host could not hold it (per-element work grows ~N/n_used)
    rate = hpsi / el
    if n_used != n:
        rate = rate * (2 ** n_used) / (2 ** n) * (n_used / n)
    return {"value": rate, "unit": "H.psi/s", "cores": int(lib.svref_threads()), "kind": "port",
            "sample": (f"C/OpenMP restatement of rydsim/_kernels.py:14 matvec at N={n_used}"
                       + ("" if n_used == n else f" scaled to N={n}")
                       + f", {done} slices of 2^{n_used - chunk_log2} outputs ({hpsi:.3f} H.psi) in {el:.1f} s"),
            "elapsed_s": el, "n_used": n_used}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(gpus):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        # one GPU per rank; modulo only so the sharded path can be smoke-tested with several ranks on
        # a one-GPU box (RSV_BENCH_BACKEND=gloo)
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("RSV_BENCH_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
        pg = dist
    return rank, world, local, pg


def max_over_ranks(x, pg):
    if pg is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    # CPU only: rank 0 alone runs it; the other ranks exit at once (no process group, no barrier),
    # so none of them spins on a host core the reference's threads could use
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    t0 = time.time()
    steps = args.steps
    res = cpu_baseline(args.n, steps=steps, warmup=args.warmup, chunk_log2=max(0, args.n - 24))
    # second leg: the reference's own kernel as the reference runs it (numba, serial), restated in
    # oracle/numba_ref.py (identical outputs to rydsim/_kernels.py:13: profiles/r2_numba_reference.json)
    numba_leg = None
    if not args.no_numba:
        try:
            from oracle import numba_ref

            numba_leg = numba_ref.time_sample(args.n, seconds=args.numba_seconds)
            numba_leg.pop("elapsed_s", None)
        except Exception as exc:  # pragma: no cover - numba missing on the host
            numba_leg = {"value": None, "sample": f"unavailable: {exc}"}
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": res["value"], "unit": "H.psi/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * res["elapsed_s"] / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic",
        "config": {"workload": f"random{args.n}: N={args.n} random 2D register, per-atom detuning map, "
                               "1 us pulse; one step = H.psi on a bounded output slice",
                   "n_qubits": args.n},
        "cpu_baseline": {"value": res["value"], "unit": "H.psi/s", "cores": res["cores"], "kind": "port",
                         "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": "H.psi/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_numba": numba_leg,
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
NCU_SUMMARIES = ("r2_ncu_n29_final.json",            # round-2 HEAD: lo (256 threads), mid, last, combine
                 "r2_ncu_n29_last_tstore.json",      # the last pass as it is now (TMA stores, round 2)
                 "r2_ncu_n29_before_tstore.json",    # lo / mid / combine (unchanged since)
                 "r1_ncu_n29_summary.json")


def ncu_traffic(family, n, plan):
    """DRAM bytes per launch of `family` from the newest committed ncu --set full summary
    (profiles/) that captured this N, pass plan and kernel family; else None."""
    for name in NCU_SUMMARIES:
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                d = json.load(fh)
        except Exception:
            continue
        if d.get("n") != n or d.get("plan", "plain") != plan:
            continue
        k = d.get("kernels", {}).get(family)
        if k and "traffic_bytes" in k:
            return int(k["traffic_bytes"]), k.get("kernel"), name
    return None, None, None


def alg_bytes_per_launch(family, n, k_avg, diag):
    """Algorithmic HBM bytes of one launch of a kernel family ('Roofline accounting').

    iter2: lo + last in one launch (fused two-pass iteration)
    lo   : read s_j (16 B) + s_{j-1} (16 B, all but the first iteration of a step) + write u (16 B)
           (+ 8 B of precomputed diagonal for diag='vec')
    chunk: the same bytes for two bit groups (its second tile pass re-reads s_j and u' from L2)
    mid  : read s_j + u, write u            (48 B)
    last : read s_j + u, write s_{j+1}      (48 B)
    combine : read the k basis vectors, write psi ((k + 1) x 16 B)
    """
    amp = 2 ** n
    if family == "iter2":   # fused [lo, last] iteration (13..21 qubits): both passes' bytes
        prev_frac = (k_avg - 1.0) / k_avg if k_avg > 0 else 0.0
        return (32 + 16 * prev_frac + (8 if diag == "vec" else 0) + 48) * amp
    if family in ("lo", "chunk", "first"):
        prev_frac = (k_avg - 1.0) / k_avg if k_avg > 0 else 0.0
        return (32 + 16 * prev_frac + (8 if diag == "vec" else 0)) * amp
    if family in ("mid", "last"):
        return 48 * amp
    return (k_avg + 1) * 16 * amp


def run_sharded(args, rank, world, local, pg):
    """--gpus P > 1: one shard per GPU (row e), weak scaling: N = n + log2(P) qubits, 2^n amplitudes
    per GPU. Local bit-group passes + global-qubit exchanges (NCCL P2P, the first overlapped with the
    local passes) + all-reduced Lanczos scalars. value counts N=n-equivalent products (x 2^(N-n)), so
    perfect weak scaling gives P x the one-GPU value."""
    import torch
    import torch.distributed as dist

    from paper_2510_09813_b200 import KrylovConfig, interaction_matrix, workloads
    from paper_2510_09813_b200.sharding import FusedShardEngine, evolve_sv_sharded_fused

    n_glob = int(math.log2(world))
    strong = args.total_qubits is not None   # BASELINE configs[4]: fixed N (e.g. 33) over P GPUs
    n_tot = args.total_qubits if strong else args.n + n_glob
    if strong:
        args.n = n_tot - n_glob
    reg, seq = workloads.config(args.workload, dt_ns=args.dt, n_override=n_tot)
    total_steps = args.warmup + args.steps
    cfg = KrylovConfig(args.tol)
    u = interaction_matrix(reg)
    t_setup = time.time()
    eng = FusedShardEngine(n_tot, u, dist, device=torch.device("cuda", local), max_krylov_dim=cfg.max_krylov_dim,
                           peer_memory=not args.no_peer_memory, krylov_vectors_cap=args.krylov_cap)
    peer_mode = eng.peer_memory
    stream = torch.cuda.current_stream()

    def do_step(k):
        nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
        return eng.step(*seq.step(k), float(seq.dt_ns), cfg.tolerance, cfg.max_krylov_dim, next_params=nxt,
                        observe=True)

    w0 = torch.cuda.Event(enable_timing=True)
    w1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0.record(stream)
    for k in range(args.warmup):
        do_step(k)
    w1.record(stream)
    torch.cuda.synchronize()
    warm_ms = max_over_ranks(w0.elapsed_time(w1), pg)
    barrier(pg)
    eng.eng.set_profiling(True)
    sampler = ClockSampler(local)
    sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    reps = [do_step(k) for k in range(args.warmup, total_steps)]
    occ = eng.occupations()   # host read of the step's result (all-reduced)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(pg)
    ms = max_over_ranks(ev0.elapsed_time(ev1), pg)
    prof = eng.eng.profile()
    matvecs = sum(r.matvecs for r in reps)
    iters = [r.iterations for r in reps]
    secs = ms / 1e3
    scale = 1 if strong else 2 ** (n_tot - args.n)
    value = matvecs * scale / secs
    fam = max(prof, key=lambda f: prof[f]["ms"])
    k_avg = float(np.mean(iters)) if iters else 1.0
    avg_launch_ms = prof[fam]["ms"] / max(1, prof[fam]["launches"])
    alg = alg_bytes_per_launch(fam, args.n, k_avg, "fly")
    achieved = alg / (avg_launch_ms / 1e3) / 1e9
    hbm_peak, peak_kind = peaks()
    krylov_cap = eng.eng.krylov_cap
    peer_passes = eng.peer_stats()
    eng.close()
    del eng
    torch.cuda.ipc_collect()
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:   # public API, host shard in (pinned) and out
        host_in = torch.zeros(2 ** args.n, dtype=torch.complex128, pin_memory=True)
        if rank == 0:
            host_in[0] = 1.0
        host_out = torch.empty(2 ** args.n, dtype=torch.complex128, pin_memory=True)
        sub = type(seq)(seq.dt_ns, seq.omegas[:total_steps], seq.deltas[:total_steps], seq.dt_ns * total_steps)
        torch.cuda.synchronize()
        barrier(pg)
        t0 = time.perf_counter()
        psi, reps2, _occ = evolve_sv_sharded_fused(sub, reg, dist, tolerance=cfg.tolerance,
                                                   device=torch.device("cuda", local), initial_local=host_in,
                                                   peer_memory=not args.no_peer_memory,
                                                   krylov_vectors_cap=args.krylov_cap)
        host_out.copy_(psi)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t0), pg)
        mv2 = sum(r.matvecs for r in reps2)
        e2e = {"value": mv2 * scale / (e2e_ms / 1e3), "unit": "H.psi/s",
               "h2d_bytes_per_step": int(16 * 2 ** args.n / total_steps),
               "d2h_bytes_per_step": int((16 * 2 ** args.n + 8 * n_tot * total_steps) / total_steps),
               "steps": total_steps, "ms": e2e_ms,
               "path": "paper_2510_09813_b200.sharding.evolve_sv_sharded_fused(host shard in) + shard copied out"}
        del psi
        torch.cuda.empty_cache()
    pulse_us = seq.dt_ns * seq.step_count / 1000.0
    if total_steps == seq.step_count:
        pulse_fields = {"s_per_us_pulse": (warm_ms + ms) / 1e3 / pulse_us,
                        "pulse_measured_s": {"device": (warm_ms + ms) / 1e3, "steps": total_steps,
                                             "e2e": (e2e["ms"] / 1e3) if e2e else None}}
    else:
        pulse_fields = {"s_per_us_pulse_extrapolated": ms / args.steps * seq.step_count / 1e3 / pulse_us,
                        "pulse_measured_s": None}
    # self-check of the multi-GPU run: the communicator saw every rank, one GPU per rank, and the mode
    # (peer memory: TMA ring or P2P loads; or exchange) that actually ran
    devs = [None] * world
    props = torch.cuda.get_device_properties(local)
    dist.all_gather_object(devs, (torch.cuda.current_device(), str(getattr(props, "uuid", local))))
    mg_check = {"backend": dist.get_backend(), "world": dist.get_world_size(), "requested": args.gpus,
                "distinct_gpus": len({d[1] for d in devs}), "peer_memory": bool(peer_mode),
                "peer_passes": peer_passes,   # partner tiles by TMA ring / per-thread P2P loads
                "ok": dist.get_world_size() == args.gpus}
    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": value, "unit": "H.psi/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic",
            "config": {
                "workload": f"random{n_tot}: N={n_tot} random 2D register sharded by the top {n_glob} qubits "
                            f"over {world} GPUs (2^{args.n} amplitudes per GPU), per-atom detuning map, "
                            f"1 us pulse, dt={args.dt} ns, Krylov tol {args.tol}",
                "n_qubits": n_tot, "n_local": args.n, "dt_ns": args.dt, "pulse_steps": seq.step_count,
                "timed_steps": f"{args.warmup + 1}..{total_steps}", "diag": "fly",
                "parallelism": (f"{world} shards (top-qubit sharding; global-qubit flips by "
                                + ("P2P loads of the partner shards (CUDA IPC peer mappings)" if peer_mode
                                   else f"{dist.get_backend()} exchange") + f"; {dist.get_backend()} all-reduce)"),
                "value_units": (f"H.psi of the N={n_tot} register" if strong
                                else f"N={args.n}-equivalent H.psi: products x 2^(N - {args.n})"),
                "l2": "inputs larger than L2 (shard = %.1f GB)" % (16 * 2 ** args.n / 1e9),
                "krylov_vectors_resident": krylov_cap,
            },
            **pulse_fields,
            "multi_gpu_check": mg_check,
            "krylov": {"iterations_mean": k_avg, "iterations_max": max(iters) if iters else 0,
                       "matvecs": matvecs, "substeps": sum(r.substeps for r in reps)},
            "kernel_ms": {f: round(v["ms"], 3) for f, v in prof.items()},
            "roofline": {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": hbm_peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": None,
                         "alg_bytes_per_launch": alg, "avg_launch_ms": avg_launch_ms},
            "gpu_launches": int(sum(v["launches"] for v in prof.values())),
            "clocks": clocks, "e2e": e2e, "cpu_baseline": None,
            "final_occupations": [round(float(x), 6) for x in occ],
            "job_wall_s": round(time.time() - t_setup, 1),   # whole job incl. the e2e leg
        }
        print(json.dumps(line), flush=True)
    barrier(pg)
    return 0


def run_ours(args):
    import torch

    rank, world, local, pg = dist_setup(args.gpus)
    if world > 1 and not args.replicas:
        return run_sharded(args, rank, world, local, pg)
    from paper_2510_09813_b200 import KrylovConfig, ObservableSpec, SvRunConfig, evolve_sv, interaction_matrix
    from paper_2510_09813_b200 import workloads
    from paper_2510_09813_b200.engine import SvEngine

    n = args.n
    reg, seq = workloads.config(args.workload, dt_ns=args.dt, n_override=n)
    total_steps = args.warmup + args.steps
    if total_steps > seq.step_count:
        raise SystemExit(f"warmup+steps={total_steps} exceeds the {seq.step_count}-step pulse")
    cfg = KrylovConfig(args.tol)
    u = interaction_matrix(reg)
    t_setup = time.time()
    eng = SvEngine(n, u, diag=args.diag, max_krylov_dim=cfg.max_krylov_dim)
    if args.plan_gm != -1:
        eng.set_plan(args.plan_gm)
    eng.set_observables([1 << q for q in range(n)])
    plan = eng.pass_plan()
    stream = torch.cuda.current_stream()

    def do_step(k):
        nxt = seq.step(k + 1) if k + 1 < seq.step_count else None
        om, de = seq.step(k)
        rep = eng.step(om, de, float(seq.dt_ns), cfg.tolerance, cfg.max_krylov_dim, cfg.norm_epsilon,
                       next_params=nxt, observe=True)
        occ = eng.observables()   # device -> host read of the step's result
        return rep, occ

    w0 = torch.cuda.Event(enable_timing=True)
    w1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0.record(stream)
    for k in range(args.warmup):
        do_step(k)
    w1.record(stream)
    torch.cuda.synchronize()
    warm_ms = max_over_ranks(w0.elapsed_time(w1), pg)
    barrier(pg)
    # per-kernel CUDA events around every launch at N >= 24; on smaller registers (host-paced ~35 us
    # Lanczos iterations) every 16th launch per kernel family, the event pairs otherwise slow the
    # timed loop itself (configs[1]: 16 %, tools/l20_overhead.py)
    prof_every = 1 if n >= 24 else 16
    eng.set_profiling(True, every=prof_every)
    sampler = ClockSampler(local)
    sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    reps = []
    for k in range(args.warmup, total_steps):
        rep, occ = do_step(k)
        reps.append(rep)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(pg)
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local, pg)
    prof = eng.profile()
    matvecs = sum(r.matvecs for r in reps)
    iters = [r.iterations for r in reps]
    substeps = sum(r.substeps for r in reps)
    krylov_cap = eng.krylov_cap
    final_occ = occ.tolist()

    secs = ms / 1e3
    value = world * matvecs / secs
    ms_per_step = ms / args.steps
    hbm_peak, peak_kind = peaks()
    eff_gbs = world * matvecs * 32 * 2 ** n / secs / 1e9
    # dominant kernel family by device time inside the timed region
    fam = max(prof, key=lambda f: prof[f]["ms"])
    launches = prof[fam]["launches"]
    k_avg = float(np.mean(iters)) if iters else 1.0
    avg_launch_ms = prof[fam]["ms"] / max(1, launches)
    alg = alg_bytes_per_launch(fam, n, k_avg, args.diag)
    achieved = alg / (avg_launch_ms / 1e3) / 1e9
    kernel_launches = int(sum(v["launches"] for v in prof.values()))
    plan_name = "chunk" if plan and plan[0].get("family") == "chunk" else "plain"
    traffic, traffic_kernel, traffic_file = (ncu_traffic(fam, n, plan_name) if args.diag == "fly"
                                               else (None, None, None))
    pass_ms = {f: round(v["ms"], 3) for f, v in prof.items()}

    # the rest of the pulse after the timed steps (outside the timed region of `value`), so the
    # whole 1 us pulse is always measured on the device: warm-up + timed + rest steps
    rest_ms = 0.0
    if total_steps < seq.step_count and not args.no_rest:
        eng.set_profiling(False)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        r0.record(stream)
        for k in range(total_steps, seq.step_count):
            do_step(k)
        r1.record(stream)
        torch.cuda.synchronize()
        rest_ms = max_over_ranks(r0.elapsed_time(r1), pg)

    # ---- e2e through the public API: host initial state in, host final state + occupations out
    e2e = None
    if not args.no_e2e:
        # the engine's blocks go back to torch's caching allocator, where evolve_sv's own engine
        # finds them (no empty_cache: re-allocating the Krylov workspace from the driver cost
        # ~0.5 s per call at configs[1], more than its whole 3 us sweep)
        del eng
        host_in = torch.zeros(2 ** n, dtype=torch.complex128, pin_memory=True)
        host_in[0] = 1.0
        host_out = torch.empty(2 ** n, dtype=torch.complex128, pin_memory=True)
        sub = type(seq)(seq.dt_ns, seq.omegas[:total_steps], seq.deltas[:total_steps], seq.dt_ns * total_steps)
        torch.cuda.synchronize()
        barrier(pg)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        res = evolve_sv(sub, reg, SvRunConfig(krylov=cfg, initial_state=host_in,
                                              observables=(ObservableSpec("occupation", (), 1),),
                                              diag=args.diag, allow_above_cap=True))
        host_out.copy_(res.final_state, non_blocking=False)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * wall), pg)
        mv = sum(r.matvecs for r in res.krylov_reports)
        state_bytes = 16 * 2 ** n
        e2e = {"value": world * mv / (e2e_ms / 1e3), "unit": "H.psi/s",
               "h2d_bytes_per_step": int((state_bytes + 16 * n * total_steps) / total_steps),
               "d2h_bytes_per_step": int((state_bytes + 8 * n * total_steps) / total_steps),
               "steps": total_steps, "ms": e2e_ms,
               "path": "paper_2510_09813_b200.evolve_sv(host initial state) + final state copied to pinned host"}
        del res
        torch.cuda.empty_cache()

    # s per 1 us pulse: measured only when warm-up + timed steps are the whole pulse (device time of
    # all of its steps); otherwise an extrapolation from the timed steps, named as such
    pulse_us = seq.dt_ns * seq.step_count / 1000.0
    pulse_fields = {}
    if total_steps == seq.step_count:
        pulse_fields["s_per_us_pulse"] = (warm_ms + ms) / 1e3 / pulse_us
        pulse_fields["pulse_measured_s"] = {"device": (warm_ms + ms) / 1e3,
                                            "e2e": (e2e["ms"] / 1e3) if e2e else None,
                                            "steps": total_steps}
    elif rest_ms > 0.0:   # warm-up + timed steps, then the rest of the pulse: all of it measured
        pulse_fields["s_per_us_pulse"] = (warm_ms + ms + rest_ms) / 1e3 / pulse_us
        pulse_fields["pulse_measured_s"] = {"device": (warm_ms + ms + rest_ms) / 1e3, "e2e": None,
                                            "steps": seq.step_count,
                                            "split": {"warmup": args.warmup, "timed": args.steps,
                                                      "rest": seq.step_count - total_steps}}
    else:
        pulse_fields["s_per_us_pulse_extrapolated"] = ms_per_step * seq.step_count / 1e3 / pulse_us
        pulse_fields["pulse_measured_s"] = None
    # per-H.psi roofline: the irreducible 48 B/amp of a Lanczos iteration (read v_j, v_{j-1}, write w)
    # over the device time of its passes (every family but the Krylov combination)
    pass_total_ms = sum(v["ms"] for f, v in prof.items() if f != "combine")
    irreducible = 48.0 * 2 ** n * matvecs
    per_hpsi = {"irreducible_bytes_per_amp": 48, "iteration_ms": pass_total_ms / max(1, matvecs),
                "achieved_gbs": irreducible / (pass_total_ms / 1e3) / 1e9 if pass_total_ms else None,
                "frac": (irreducible / (pass_total_ms / 1e3) / 1e9 / hbm_peak) if pass_total_ms else None,
                "passes_bytes_per_amp": 48 * (len(plan) if plan else 1)}
    # the plan's own bound: its passes move passes_bytes_per_amp, so at the copy peak the per-H.psi
    # fraction cannot exceed 48 / passes_bytes_per_amp
    per_hpsi["plan_bound_frac"] = 48.0 / per_hpsi["passes_bytes_per_amp"]
    per_hpsi["frac_of_plan_bound"] = (per_hpsi["frac"] / per_hpsi["plan_bound_frac"]
                                      if per_hpsi["frac"] is not None else None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(n, seconds=args.cpu_seconds)
            cpu.pop("elapsed_s", None)
            cpu.pop("n_used", None)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "H.psi/s", "cores": None, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": BASELINE_METRIC,
            "value": value,
            "unit": "H.psi/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "complex128 (f64)",
            "data": "synthetic",
            "config": {
                "workload": f"{args.workload}: N={n} " + WORKLOAD_TEXT.get(args.workload, args.workload)
                            + f", dt={args.dt} ns, Krylov tol {args.tol}",
                "n_qubits": n, "dt_ns": args.dt, "pulse_steps": seq.step_count,
                "timed_steps": f"{args.warmup + 1}..{total_steps}",
                "diag": args.diag,
                "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                "l2": ("inputs larger than L2 (state = %.1f GB)" % (16 * 2 ** n / 1e9)
                       if 3 * 16 * 2 ** n > 126e6 else
                       "no flush: the state (%.1f MB) and an iteration's three vectors fit in the 126 MB L2 -- the "
                       "configuration's own working set; the step's Krylov basis (%d vectors on average) does not"
                       % (16 * 2 ** n / 1e6, round(k_avg))),
                "kernel_timing": ("CUDA events around every launch" if prof_every == 1 else
                                  f"CUDA events around every {prof_every}th launch per kernel family (mean x launches)"),
                "pass_plan": plan,
                "krylov_vectors_resident": krylov_cap,
            },
            "hbm_gbs_effective": eff_gbs,
            **pulse_fields,
            "krylov": {"iterations_mean": k_avg, "iterations_max": max(iters) if iters else 0,
                       "matvecs": matvecs, "substeps": substeps},
            "kernel_ms": pass_ms,
            "roofline": {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": hbm_peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": traffic,
                         "traffic_source": (f"profiles/{traffic_file} (dram__bytes_read.sum + "
                                            f"dram__bytes_write.sum of one {traffic_kernel} launch)"
                                            if traffic else None),
                         "alg_bytes_per_launch": alg, "avg_launch_ms": avg_launch_ms},
            "per_hpsi": per_hpsi,
            "gpu_launches": kernel_launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "final_occupations": [round(x, 6) for x in final_occ],
            "job_wall_s": round(time.time() - t_setup, 1),   # whole job incl. the e2e and CPU legs
        }
        print(json.dumps(line), flush=True)
    barrier(pg)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=97)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=29)
    ap.add_argument("--workload", default="random29")
    ap.add_argument("--dt", type=int, default=10)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--diag", default="fly", choices=["fly", "vec"])
    ap.add_argument("--plan-gm", type=int, default=-1,
                    help="pass plan: -1 auto, 0 plain bit-group passes, 3..9 L2 chunk pass (A/B runs)")
    ap.add_argument("--total-qubits", type=int, default=None,
                    help="N > 1: strong scaling of a fixed register (BASELINE configs[4]: 33) instead of n + log2 P")
    ap.add_argument("--krylov-cap", type=int, default=None,
                    help="N > 1: resident Krylov vectors per rank (default: what fits; smoke runs of several "
                         "ranks on one GPU need a cap)")
    ap.add_argument("--no-peer-memory", action="store_true",
                    help="N > 1: exchange the partner shards' vectors instead of reading them over NVLink")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent N=--n replicas instead of one sharded N + log2(P) register")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rest", action="store_true",
                    help="do not run the rest of the pulse after the timed steps (no measured pulse time)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-numba", action="store_true", help="--impl reference: skip the serial numba leg")
    ap.add_argument("--numba-seconds", type=float, default=10.0)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("note: warm-up < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
