#!/bin/bash
# round-2 GPU call B: new regen/speculation tests, TMA de-interleave micro-benchmark, bench (N=29, lattice20)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "regeneration or speculative or substepping or host_final or reference_diagonal or build_diagonal" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest.log
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pb tools/plane_tma_bench.cu -lcuda && timeout 300 /tmp/pb > gpurun_out/r2b_plane_tma.txt 2>&1; echo "pb rc=$?"; cat gpurun_out/r2b_plane_tma.txt
timeout 900 python bench.py --no-cpu > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload lattice20 --qubits 20 --steps 297 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2b_l20.json 2> gpurun_out/r2b_l20.err; echo "l20 rc=$?"
