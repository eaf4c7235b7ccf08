#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/stepprof.py 29 70 1 -1 -1 30 > gpurun_out/r2d_prof_regen.txt 2>&1; echo rc=$?
timeout 900 python tools/stepprof.py 29 70 0 -1 -1 30 > gpurun_out/r2d_prof_split.txt 2>&1; echo rc=$?
tail -1 gpurun_out/r2d_prof_regen.txt; tail -1 gpurun_out/r2d_prof_split.txt
