#!/bin/bash
# Full GPU suite (no -x) + configs[2] lattice27 and configs[1] lattice20 bench lines at HEAD.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2t_pytest.log
timeout 900 python bench.py --workload lattice27 --n 27 --no-cpu > gpurun_out/r2t_l27.json 2> gpurun_out/r2t_l27.err; echo "l27 rc=$?"
timeout 600 python bench.py --workload lattice20 --n 20 --steps 297 --warmup 3 --no-cpu > gpurun_out/r2t_l20.json 2> gpurun_out/r2t_l20.err; echo "l20 rc=$?"
