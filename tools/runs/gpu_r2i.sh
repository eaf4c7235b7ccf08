#!/bin/bash
# TMA-store / transposed q-sweep: parity subset, then per-pass A/B at N=29 on one box
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity_gpu.py -x -q -k "not full_sweep and not lanczos_steps" > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2i_pytest.log
for lib in default tools/_rsv_old.so tools/_rsv_qt.so default tools/_rsv_old.so; do
  if [ $lib = default ]; then timeout 300 python tools/passbench.py 29 3; else RSV_LIB=$lib timeout 300 python tools/passbench.py 29 3; fi
done > gpurun_out/r2i_passbench.json 2>&1; cat gpurun_out/r2i_passbench.json
