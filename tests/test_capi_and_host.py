"""CPU checks: the C-ABI library loads and exports every symbol include/rsv.h declares;
host-side mirror logic (registers, pulses, configs, estimates) matches the reference semantics."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2510_09813_b200 as rs
from paper_2510_09813_b200 import _native
from paper_2510_09813_b200.errors import ConfigurationError, ValidationError

from conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "rsv.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rsv_[a-z0-9_]+)\s*\(", text)))


class TestCAbi:
    def test_library_exports_every_declared_symbol(self):
        lib = ctypes.CDLL(_native.LIB_PATH)
        syms = header_symbols()
        assert len(syms) >= 20
        for s in syms:
            assert hasattr(lib, s), s

    def test_binding_table_matches_header(self):
        assert sorted(_native.SIGNATURES) == header_symbols()

    def test_load_and_version_without_gpu(self):
        lib = _native.load()
        assert lib.rsv_version() == 10000

    def test_create_fails_loudly_without_device(self):
        import torch

        if torch.cuda.is_available():
            pytest.skip("has a GPU")
        lib = _native.load()
        ctx = ctypes.c_void_p()
        u = np.zeros((2, 2))
        rc = lib.rsv_create(2, _native.dptr(u), 1, None, ctypes.byref(ctx))
        assert rc == _native.RSV_ERR_CUDA
        assert b"no CPU fallback" in lib.rsv_last_error() or b"CUDA" in lib.rsv_last_error()

    @pytest.mark.parametrize("k", [1, 2, 3, 7, 20, 38, 60, 120])
    def test_tridiagonal_exponential_vs_oracle(self, k):
        # host-only entry point (no GPU): the Lanczos tridiagonal exp(-i tau T) e1 of krylov.py:54 by the
        # driver's Chebyshev expansion, against the oracle's dense-eigh restatement: every component
        # (full=1, the combination coefficients) and the last one alone (full=0, the convergence test)
        from oracle import sv_oracle as O

        lib = _native.load()
        rng = np.random.default_rng(k)
        for scale, tau in ((30.0, 0.01), (1500.0, 0.01), (800.0, -0.004), (5.0, 0.0)):
            a = rng.uniform(-scale, scale, k)
            b = rng.uniform(0.1 * scale, 0.6 * scale, max(k - 1, 0))
            ref = O.tridiag_exp_e1(a, b, tau)
            out = np.zeros(2 * k)
            bp = _native.dptr(b) if k > 1 else None
            assert lib.rsv_tridiag_exp_e1(_native.dptr(a), bp, k, tau, 1, _native.dptr(out)) == 0
            full = out[0::2] + 1j * out[1::2]
            assert np.abs(full - ref).max() <= 1e-12
            last = np.zeros(2)
            assert lib.rsv_tridiag_exp_e1(_native.dptr(a), bp, k, tau, 0, _native.dptr(last)) == 0
            assert abs(complex(last[0], last[1]) - ref[-1]) <= 1e-13

    def test_product_never_imports_oracle(self):
        pkg = os.path.join(ROOT, "paper_2510_09813_b200")
        for root, _, files in os.walk(pkg):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h")):
                    src = open(os.path.join(root, f)).read()
                    assert "import oracle" not in src and "from oracle" not in src, f
                    assert "sv_oracle" not in src, f


class TestHostMirror:
    def test_register_validation(self):
        with pytest.raises(ValidationError):
            rs.Register((), 1.0)
        with pytest.raises(ValidationError):
            rs.Register(((0.0, 0.0), (0.0, 0.0, 1.0)), 1.0)
        with pytest.raises(ValidationError):
            rs.interaction_matrix(rs.Register(((1.0, 2.0), (1.0, 2.0)), 1.0))

    def test_interaction_matrix_values(self):
        u = rs.interaction_matrix(rs.Register(((0.0, 0.0), (5.0, 0.0), (10.0, 0.0)), 5_000_000.0))
        assert u[0, 1] == pytest.approx(320.0) and u[1, 2] == pytest.approx(320.0)
        assert u[0, 2] == pytest.approx(5.0) and u[0, 0] == 0.0
        g = np.load(os.path.join(GOLDEN, "evolve_detmap12.npz"))
        u = rs.interaction_matrix(rs.Register(tuple(map(tuple, g["positions"])), float(g["c6"])))
        assert np.abs(u - g["u"]).max() <= 1e-12 * np.abs(u).max()

    def test_pulses_mirror_matches_reference(self):
        g = np.load(os.path.join(GOLDEN, "pulses.npz"))
        import math

        w = rs.pulses.blackman_window(120)
        area = 2 * math.pi * w.sum() / w.max()
        prog = rs.ChannelProgram.from_channels([[rs.Blackman(120, area)] for _ in range(3)],
                                               [[rs.Ramp(120, -6 * math.pi, 4 * math.pi)] for _ in range(3)], 120)
        s = rs.sample_program(prog)
        assert np.abs(s.omega - g["adiabatic_omega"]).max() <= 1e-12
        assert np.abs(s.delta - g["adiabatic_delta"]).max() <= 1e-12
        d = rs.discretize(s, 8)
        assert np.abs(d.omegas - g["adiabatic_disc_omega_dt8"]).max() <= 1e-12
        with pytest.raises(ConfigurationError):
            rs.discretize(s, 7)

    def test_configs_and_estimates(self):
        assert rs.memory_estimate_sv(1, 1) == 96
        assert rs.memory_estimate_sv(26, 0) == 16 * 2 ** 26 * 2
        assert rs.memory_estimate_sv(26, 15) < 20e9
        with pytest.raises(ValidationError):
            rs.KrylovConfig(tolerance=0.0)
        with pytest.raises(ValidationError):
            rs.KrylovConfig(max_krylov_dim=1)
        with pytest.raises(ValidationError):
            rs.ObservableSpec("correlation", (0,))
        spec = rs.ObservableSpec("correlation", (0, 3, 1, 2))
        assert spec.masks(4) == [0b1001, 0b0110]
        assert rs.ObservableSpec("occupation").masks(3) == [1, 2, 4]

    def test_slice_validation(self):
        with pytest.raises(ValidationError):
            rs.HamiltonianSlice(np.zeros(2), np.zeros(3))
        with pytest.raises(ValidationError):
            rs.HamiltonianSlice.from_parameters([1.0, 2.0], [0.0], np.zeros((2, 2)))
        s = rs.HamiltonianSlice.from_parameters([1.0, 2.0], [0.5, 0.0], np.zeros((2, 2)))
        assert s.structured and s.qubit_count == 2
