#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_iteration or speculative" > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2r_pytest.log
for i in 1 2; do timeout 600 python bench.py --workload lattice20 --n 20 --steps 297 --warmup 3 --no-cpu > gpurun_out/r2r_l20_$i.json 2> gpurun_out/r2r_l20_$i.err; echo "l20 rc=$?"; done
