#!/bin/bash
mkdir -p gpurun_out
for v in default it512; do
  if [ $v = default ]; then unset RSV_LIB; else export RSV_LIB=$PWD/tools/_rsv_$v.so; fi
  for i in 1 2; do
    timeout 600 python bench.py --workload lattice20 --qubits 20 --steps 297 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2z_${v}_$i.json 2> gpurun_out/r2z_${v}_$i.err; echo "$v $i rc=$?"
  done
done
