set -x
timeout 600 python -m pytest tests/test_chunk_pass.py -x -q 2>&1 | tail -3
pb() { timeout 300 python tools/passbench.py 29 4; }
RSV_PLAN_GM=0 pb
pb
RSV_PLAN_GM=9 pb
RSV_PLAN_GM=9 RSV_PLAN_LAG=512 pb
RSV_PLAN_GM=9 RSV_PLAN_LAG=1024 pb
RSV_LIB=tools/_rsv_nodeleg.so pb
RSV_LIB=tools/_rsv_nodeleg.so RSV_PLAN_GM=9 pb
RSV_LIB=tools/_rsv_nohints.so RSV_PLAN_GM=9 pb
