#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q  > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2p_pytest.log
timeout 600 python bench.py --workload lattice20 --n 20 --steps 297 --warmup 3 --no-cpu > gpurun_out/r2p_l20.json 2> gpurun_out/r2p_l20.err; echo "l20 rc=$?"
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "bench rc=$?"
