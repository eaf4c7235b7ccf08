"""TEST INFRASTRUCTURE ONLY -- the reference's compiled matvec as the reference compiles it.

rydsim/_kernels.py:13 ``matvec_bitflip_diag`` is a numba ``@njit(cache=True)`` loop (serial: no
``parallel=True``), dispatched by hamiltonian.py:180-187 for N >= 10. This restates that loop for
numba on the GPU box's host, where /root/reference does not exist, so ``bench.py --impl
reference`` can time the reference's own single-threaded kernel beside the OpenMP C port
(``oracle/sv_ref.c``). The only change is the output range [b0, b1) (a bounded sample of one
H.psi; every element still reads its N partners across the whole state). tools/numba_reference.py
checks, in the build container, that this restatement and the real rydsim kernel give identical
outputs and the same time per element.
"""

import numpy as np
from numba import njit


@njit(cache=True)
def matvec_bitflip_diag_range(psi, diag, half_omega, out, b0, b1):
    nq = half_omega.shape[0]
    for b in range(b0, b1):
        acc = diag[b] * psi[b]
        for i in range(nq):
            c = half_omega[i]
            if c != 0.0:
                acc += c * psi[b ^ (1 << i)]
        out[b] = acc


def time_sample(n, seconds=10.0, slice_log2=20, seed=3):
    """H.psi/s of the serial numba kernel at N=n on 2^slice_log2-output slices (bounded sample)."""
    import time

    rng = np.random.default_rng(seed)
    dim = 1 << n
    psi = np.empty(dim, dtype=np.complex128)
    step = 1 << 22
    for b in range(0, dim, step):   # no 2^n-sized temporaries
        m = min(step, dim - b)
        psi[b:b + m].real = rng.standard_normal(m)
        psi[b:b + m].imag = rng.standard_normal(m)
    diag = rng.uniform(-10.0, 10.0, dim)
    half = 0.5 * rng.uniform(0.5, 4.0, n)
    out = np.empty_like(psi)
    sl = 1 << min(slice_log2, n)
    matvec_bitflip_diag_range(psi, diag, half, out, 0, 64)   # compile outside the timed region
    t0 = time.perf_counter()
    done = 0
    while True:
        b0 = (done * sl) % dim
        matvec_bitflip_diag_range(psi, diag, half, out, b0, b0 + sl)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": done * sl / dim / el, "unit": "H.psi/s", "cores": 1, "kind": "port",
            "sample": (f"numba restatement of rydsim/_kernels.py:13 (serial @njit, as the reference runs it) "
                       f"at N={n}, {done} slices of 2^{min(slice_log2, n)} outputs in {el:.1f} s"),
            "elapsed_s": el}
