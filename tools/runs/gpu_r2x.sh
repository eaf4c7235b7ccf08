#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharding_fused_gpu.py -q -x > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2x_pytest.log
for mode in 1 0; do
  RSV_PEER_TMA=$mode RSV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --qubits 26 --krylov-cap 8 --steps 6 --warmup 3 \
    --no-cpu --no-e2e > gpurun_out/r2x_peer$mode.json 2> gpurun_out/r2x_peer$mode.err; echo "peer$mode rc=$?"
  RSV_PEER_TMA=$mode RSV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 --qubits 25 --krylov-cap 6 --steps 6 --warmup 3 \
    --no-cpu --no-e2e > gpurun_out/r2x_peer4_$mode.json 2> gpurun_out/r2x_peer4_$mode.err; echo "peer4_$mode rc=$?"
done
