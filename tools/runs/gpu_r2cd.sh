#!/bin/bash
# tile pacing A/B at N=29 (RSV_PACE window W in tiles per CTA; default build = off), alternating runs
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2cd_smi.txt 2>&1
run() { timeout 240 python bench.py --no-cpu --no-e2e > gpurun_out/r2cd_$TAG.json 2> gpurun_out/r2cd_$TAG.err; echo "$TAG rc=$?"; }
for i in 1 2; do
  unset RSV_LIB; TAG=def$i run
  for v in pace4 pace16 pace64; do export RSV_LIB=$PWD/tools/_rsv_$v.so; TAG=$v$i run; done
done
