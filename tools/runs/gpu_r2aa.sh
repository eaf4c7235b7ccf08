#!/bin/bash
# plain 3-pass plan vs the L2 chunk pass (lo + mid in one launch, 96 B/amp) with the round-2 kernels
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --no-e2e "$@" > gpurun_out/r2aa_$TAG.json 2> gpurun_out/r2aa_$TAG.err; echo "$TAG rc=$?"; }
TAG=plain run
TAG=gm9 run --plan-gm 9
TAG=gm8 run --plan-gm 8
RSV_LIB=$PWD/tools/_rsv_nodel.so TAG=gm9nodel run --plan-gm 9
TAG=plain2 run
