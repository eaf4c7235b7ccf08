#!/bin/bash
# 2 ranks on one GPU (CUDA IPC 'peers'): TMA ring vs per-thread loads, per-pass times
mkdir -p gpurun_out
for mode in 1 0; do
  RSV_PEER_TMA=$mode RSV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --qubits 26 --krylov-cap 8 --steps 6 --warmup 3 \
    --no-cpu --no-e2e > gpurun_out/r2w_peer$mode.json 2> gpurun_out/r2w_peer$mode.err; echo "peer$mode rc=$?"
  tail -c 1500 gpurun_out/r2w_peer$mode.json
done
