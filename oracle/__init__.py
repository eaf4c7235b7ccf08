"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference (rydsim) state-vector path.

This package is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl reference``
leg may import it. The product path (``paper_2510_09813_b200``) must never
import, link or execute anything under ``oracle/``; it fails loudly when the
CUDA extension is missing instead of falling back to this code.

Contents
--------
``sv_oracle``    numpy restatement of rydsim's hamiltonian / krylov / sv / observables
                 / pulses / generator functions (each function cites the reference
                 file:line it follows).
``sv_ref.c``     plain-C (OpenMP) restatement of the reference's compiled hot loop
                 (``rydsim/_kernels.py:13`` fused bit-flip matvec) plus the Lanczos
                 vector kernels, used only as the timed CPU baseline in ``bench.py``.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference from
``/root/reference/pkg/src`` (available only in the build container) and stores
its outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
restatement against those vectors.
"""
