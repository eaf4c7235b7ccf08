set -x
timeout 600 python -m pytest tests/test_chunk_pass.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for gm in 0 -1; do for lib in default tools/_rsv_nohints.so; do
  if [ $lib = default ]; then RSV_PLAN_GM=$gm timeout 300 python tools/passbench.py 29 4; else RSV_LIB=$lib RSV_PLAN_GM=$gm timeout 300 python tools/passbench.py 29 4; fi
done; done
for lag in 256 512 1024; do RSV_PLAN_LAG=$lag timeout 300 python tools/passbench.py 29 4; done
