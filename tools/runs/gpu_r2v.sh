#!/bin/bash
# (1) ncu --set full of the fused iteration kernel at configs[1] (N=20); (2) 2 ranks on one GPU (CUDA IPC
# "peers"): TMA ring vs per-thread loads, per-pass times
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iter2_kernel --launch-skip 200 -c 2 \
  -o gpurun_out/r2v_iter2 -f python bench.py --workload lattice20 --n 20 --steps 20 --warmup 3 --no-cpu --no-e2e \
  > gpurun_out/r2v_iter2.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r2v_iter2.ncu-rep --page raw --csv > gpurun_out/r2v_iter2_raw.csv 2>/dev/null
ncu -i gpurun_out/r2v_iter2.ncu-rep --page details --csv > gpurun_out/r2v_iter2_details.csv 2>/dev/null
ncu -i gpurun_out/r2v_iter2.ncu-rep --page source --csv > gpurun_out/r2v_iter2_source.csv 2>/dev/null
rm -f gpurun_out/r2v_iter2.ncu-rep
for mode in 1 0; do
  RSV_PEER_TMA=$mode RSV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --qubits 26 --krylov-cap 8 --steps 6 --warmup 3 \
    --no-cpu --no-e2e > gpurun_out/r2v_peer$mode.json 2> gpurun_out/r2v_peer$mode.err; echo "peer$mode rc=$?"
  tail -c 1500 gpurun_out/r2v_peer$mode.json
done
