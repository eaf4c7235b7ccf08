timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/passbench.py 29 4
RSV_LIB=tools/_rsv_norot.so timeout 300 python tools/passbench.py 29 4
timeout 300 python tools/passbench.py 26 4
RSV_LIB=tools/_rsv_norot.so timeout 300 python tools/passbench.py 26 4
