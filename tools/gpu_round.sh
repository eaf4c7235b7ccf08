#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench, ncu launch list, one ncu --set full capture.
# usage (on the box): bash tools/gpu_round.sh TAG [what...]   what in: tests smoke bench launches full passbench
set -u
TAG=${1:-run}; shift
WHAT=${*:-tests smoke bench launches}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?";;
    smoke) timeout 300 python __graft_entry__.py --smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?";;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/${TAG}_bench.json;;
    benchvec) timeout 900 python bench.py --diag vec --no-e2e --no-cpu > gpurun_out/${TAG}_benchvec.json 2> gpurun_out/${TAG}_benchvec.err; echo "benchvec rc=$?";;
    ref) timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2>&1; echo "ref rc=$?";;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-rest > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?";;
    full) timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-pass_kernel} --launch-skip ${NCU_SKIP:-40} -c ${NCU_C:-3} -o gpurun_out/${TAG}_full -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-rest > gpurun_out/${TAG}_full.log 2>&1; echo "full rc=$?"
          ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
          ncu -i gpurun_out/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_full_details.csv 2>/dev/null;;
    passbench) for n in ${PB_N:-26 29}; do timeout 600 python tools/passbench.py $n 4; done > gpurun_out/${TAG}_passbench.json 2>&1; echo "passbench rc=$?"; cat gpurun_out/${TAG}_passbench.json;;
  esac
done
