"""The drop-in boundary used from plain C (tests/c_abi/consumer.c), as a cgo/JNI/FFI binding would:
the program links paper_2510_09813_b200/_rsv.so and the CUDA runtime, and checks H.psi against the C
restatement of the reference matvec (oracle/sv_ref.c) plus exact properties of rsv_expm_step. On a
machine without a GPU it checks that rsv_create fails loudly (no CPU fallback)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    from oracle import build as obuild
    from paper_2510_09813_b200 import _native

    ref = obuild.build()
    exe = str(tmp_path / "consumer")
    libdirs = [os.path.dirname(_native.LIB_PATH), os.path.dirname(ref), os.path.join(CUDA, "lib64")]
    cmd = ["gcc", "-O2", "-std=c11", "-o", exe, os.path.join(ROOT, "tests", "c_abi", "consumer.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           _native.LIB_PATH, ref, "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", "-fopenmp"]
    cmd += [f"-Wl,-rpath,{d}" for d in libdirs]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_consumer_builds_and_fails_loudly_without_gpu(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU (the GPU run is test_consumer_on_gpu)")
    exe = _build(tmp_path)
    out = subprocess.run([exe, "--expect-no-gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_consumer_on_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "c-abi consumer ok" in out.stdout
