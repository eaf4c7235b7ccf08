#!/bin/bash
# round-2 GPU call A: full GPU suite (minus the not-yet-generated lattice20 fixture), bench, reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -k "not full_sweep" --durations=15 > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2a_pytest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; echo "ref rc=$?"
