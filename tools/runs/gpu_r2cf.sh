#!/bin/bash
# Krylov combination with the next-but-one tile requested before the current one is consumed
# (RSV_COMBINE_AHEAD=1): parity subset with the variant, then alternating N=29 benches
mkdir -p gpurun_out
RSV_LIB=$PWD/tools/_rsv_ahead.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Evolve or Observables or Expm or Reorth" > gpurun_out/r2cf_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2cf_tests.log
run() { timeout 240 python bench.py --no-cpu --no-e2e > gpurun_out/r2cf_$TAG.json 2> gpurun_out/r2cf_$TAG.err; echo "$TAG rc=$?"; }
for i in 1 2 3; do
  unset RSV_LIB; TAG=def$i run
  export RSV_LIB=$PWD/tools/_rsv_ahead.so; TAG=ahead$i run
done
