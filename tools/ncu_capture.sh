#!/bin/bash
# ncu --set full of one Lanczos iteration's passes (lo, mid, last) and one Krylov combination at N
# (default 29) via tools/passbench.py; summaries land in gpurun_out/TAG_*.csv.
# usage: bash tools/ncu_capture.sh TAG [N]
TAG=$1; N=${2:-29}
mkdir -p gpurun_out
run() {  # name regex skip count
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c $4 \
     -o gpurun_out/${TAG}_$1 -f python tools/passbench.py $N 1 > gpurun_out/${TAG}_$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv > gpurun_out/${TAG}_$1_source.csv 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/${TAG}_$1.ncu-rep   # gpurun copies back <= 64 MiB
}
# launches per Lanczos iteration: lo, mid, last -> the 4th iteration's passes are launches 9, 10, 11
run lo "pass_kernel" 9 1
run mid "pass_kernel" 10 1
run last "pass_kernel" 11 1
run combine "combine_kernel" 3 1
