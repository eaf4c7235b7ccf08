#!/bin/bash
# tile pacing A/B, second try: the progress poll only every E tiles (RSV_PACE_EVERY)
mkdir -p gpurun_out
run() { timeout 240 python bench.py --no-cpu --no-e2e > gpurun_out/r2ce_$TAG.json 2> gpurun_out/r2ce_$TAG.err; echo "$TAG rc=$?"; }
for i in 1 2; do
  unset RSV_LIB; TAG=def$i run
  for v in pace8e8 pace32e8 pace8e4; do export RSV_LIB=$PWD/tools/_rsv_$v.so; TAG=$v$i run; done
done
