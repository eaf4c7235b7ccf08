#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "TestApplyHamiltonian or TestEvolve" > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2m_pytest.log
for lib in default tools/_rsv_noearly.so default tools/_rsv_noearly.so; do
  if [ $lib = default ]; then timeout 300 python tools/passbench.py 29 3; else RSV_LIB=$lib timeout 300 python tools/passbench.py 29 3; fi
done 2>&1 | tee gpurun_out/r2m_passbench.json
