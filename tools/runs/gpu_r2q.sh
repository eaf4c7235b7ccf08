#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_iteration or speculative or TestEvolve or lanczos" > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q_pytest.log
timeout 600 python bench.py --workload lattice20 --n 20 --steps 297 --warmup 3 --no-cpu > gpurun_out/r2q_l20.json 2> gpurun_out/r2q_l20.err; echo "l20 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 200 --csv --log-file gpurun_out/r2q_l20_launches.csv python bench.py --workload lattice20 --n 20 --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
