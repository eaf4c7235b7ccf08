#!/bin/bash
# ncu --set full of the diag="vec" lo pass with the staged diagonal tile (N=29), one launch
mkdir -p gpurun_out
RSV_DIAG=vec timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pass_kernel --launch-skip 9 -c 1 \
   -o gpurun_out/r2cc_lovec -f python tools/passbench.py 29 1 > gpurun_out/r2cc_lovec.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2cc_lovec.ncu-rep --page raw --csv > gpurun_out/r2cc_lovec_raw.csv 2>/dev/null
ncu -i gpurun_out/r2cc_lovec.ncu-rep --page details --csv > gpurun_out/r2cc_lovec_details.csv 2>/dev/null
rm -f gpurun_out/r2cc_lovec.ncu-rep
