#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_sweep" > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2g_pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
timeout 600 python tools/passbench.py 29 4 > gpurun_out/r2g_passbench.json 2>&1; cat gpurun_out/r2g_passbench.json
