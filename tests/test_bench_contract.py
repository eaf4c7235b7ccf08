"""bench.py's JSON line (the driver's contract) on small registers: the single-GPU line, the sharded
line of a two-rank torchrun (gloo, both ranks on one GPU) with its multi-GPU self-check, and the
reference arm under torchrun (rank 0 alone, every host core)."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


def _torchrun(nproc, args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", "bench.py", *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                          env={**os.environ, **(env or {})})


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--qubits", "16", "--steps", "3", "--warmup", "3", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    assert d["roofline"]["unit"] == "GB/s" and 0 < d["roofline"]["frac"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # the rest of the pulse runs after the timed steps: the whole pulse is measured
    assert d["pulse_measured_s"]["steps"] == d["config"]["pulse_steps"]
    assert d["per_hpsi"]["plan_bound_frac"] == pytest.approx(48.0 / d["per_hpsi"]["passes_bytes_per_amp"])


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_sharded_line_two_ranks():
    r = _torchrun(2, ["--gpus", "2", "--qubits", "15", "--krylov-cap", "8", "--steps", "3", "--warmup", "3",
                      "--no-cpu", "--no-e2e"], env={"RSV_BENCH_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    for k in KEYS:
        assert k in d, k
    chk = d["multi_gpu_check"]
    assert chk["ok"] and chk["world"] == 2 and chk["peer_memory"]
    assert chk["peer_passes"]["tma"] > 0   # partner tiles by the TMA ring
    assert d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.timeout(600)
def test_reference_arm_under_torchrun():   # CPU only (the reference arm never touches the GPU)
    r = _torchrun(2, ["--impl", "reference", "--gpus", "2", "--qubits", "18", "--steps", "3", "--warmup", "3",
                      "--no-numba"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    # every core of the affinity mask, not torchrun's OMP_NUM_THREADS=1
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
