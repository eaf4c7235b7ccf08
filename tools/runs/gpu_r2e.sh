#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:combine -c 200 --csv --log-file gpurun_out/r2e_combine.csv python tools/stepprof.py 29 4 1 -1 -1 60 > gpurun_out/r2e_prof.txt 2>&1; echo rc=$?
tail -5 gpurun_out/r2e_prof.txt
