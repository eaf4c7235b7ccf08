#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2y_bench.json 2> gpurun_out/r2y_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2y_ref.json 2> gpurun_out/r2y_ref.err; echo "ref rc=$?"
tail -c 600 gpurun_out/r2y_ref.json
