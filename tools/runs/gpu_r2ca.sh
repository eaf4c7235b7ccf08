#!/bin/bash
# combine kernel A/B at N=29 (alternating, same box): default cp.async ring, per-warp TMA ring, cp.async with the
# L2::256B prefetch-size hint; then the diag="vec" variant of the HEAD kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2ca_smi.txt 2>&1
run() { timeout 600 python bench.py --no-cpu --no-e2e $ARGS > gpurun_out/r2ca_$TAG.json 2> gpurun_out/r2ca_$TAG.err; echo "$TAG rc=$?"; }
for i in 1 2; do
  unset RSV_LIB; ARGS= TAG=def$i run
  export RSV_LIB=$PWD/tools/_rsv_ctma.so; ARGS= TAG=ctma$i run
  export RSV_LIB=$PWD/tools/_rsv_pf256.so; ARGS= TAG=pf256$i run
done
unset RSV_LIB; ARGS="--diag vec" TAG=vec run
