#!/bin/bash
mkdir -p gpurun_out
for lib in default tools/_rsv_old.so tools/_rsv_tsall.so; do
  if [ $lib = default ]; then timeout 300 python tools/dbg_apply.py 20 21 22 23; else RSV_LIB=$lib timeout 300 python tools/dbg_apply.py 20 21 22 23; fi
done > gpurun_out/r2j_dbg.txt 2>&1; cat gpurun_out/r2j_dbg.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity_gpu.py -x -q -k "not full_sweep" > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2j_pytest.log
timeout 300 python tools/passbench.py 29 3
