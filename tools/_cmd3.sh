pb() { timeout 300 python tools/passbench.py 29 4; }
for v in t256 t1024; do
  echo "== $v"
  RSV_LIB=tools/_rsv_$v.so timeout 600 python -m pytest tests/test_chunk_pass.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
  for gm in 0 -1 9; do RSV_LIB=tools/_rsv_$v.so RSV_PLAN_GM=$gm pb; done
done
echo "== default"; for gm in 0 -1; do RSV_PLAN_GM=$gm pb; done
