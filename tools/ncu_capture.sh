#!/bin/bash
# ncu --set full of one launch of each hot kernel at N (default 29) via tools/passbench.py.
# usage: bash tools/ncu_capture.sh TAG [N]
TAG=$1; N=${2:-29}
mkdir -p gpurun_out
for K in chunk_kernel pass_kernel_tma combine_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 6 -c 1 \
     -o gpurun_out/${TAG}_${K} -f python tools/passbench.py $N 1 > gpurun_out/${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
  ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page source --csv > gpurun_out/${TAG}_${K}_source.csv 2>/dev/null
done
