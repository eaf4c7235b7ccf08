#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --workload lattice20 --n 20 --steps 297 --warmup 3 --no-cpu > gpurun_out/r2o_l20.json 2> gpurun_out/r2o_l20.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2o_l20.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 300 --csv --log-file gpurun_out/r2o_l20_launches.csv python bench.py --workload lattice20 --n 20 --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
