#!/bin/bash
# diag="vec" tile staged in shared memory (RSV_DVEC_SMEM): vec-mode parity first, then the whole GPU suite,
# then the N=29 bench in both diagonal modes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vec" > gpurun_out/r2cb_vec_tests.log 2>&1; echo "vec tests rc=$?"; tail -3 gpurun_out/r2cb_vec_tests.log
timeout 900 python bench.py --no-cpu --no-e2e --diag vec > gpurun_out/r2cb_vec.json 2> gpurun_out/r2cb_vec.err; echo "vec bench rc=$?"
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2cb_fly.json 2> gpurun_out/r2cb_fly.err; echo "fly bench rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2cb_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2cb_pytest.log
