#!/bin/bash
# full GPU suite (minus the lattice20 full-sweep fixture test), smoke, ncu of the new last pass
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_sweep" > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2l_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2l_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2l_smoke.log
TAG=r2l
run() {
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c $4 \
     -o gpurun_out/${TAG}_$1 -f python tools/passbench.py 29 1 > gpurun_out/${TAG}_$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${TAG}_$1_source.csv.gz
  rm -f gpurun_out/${TAG}_$1.ncu-rep
}
run last "pass_kernel" 11 1
