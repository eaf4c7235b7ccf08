#!/bin/bash
# final: full GPU suite, smoke, default bench, configs[2] bench
mkdir -p gpurun_out
bash tools/gpu_round.sh r2ak tests smoke bench
timeout 900 python bench.py --workload lattice27 --qubits 27 --no-cpu > gpurun_out/r2ak_l27.json 2> gpurun_out/r2ak_l27.err; echo "l27 rc=$?"
