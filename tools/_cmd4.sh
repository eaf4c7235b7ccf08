RSV_LIB=tools/_rsv_lolast.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/passbench.py 29 4
RSV_LIB=tools/_rsv_lolast.so timeout 300 python tools/passbench.py 29 4
RSV_LIB=tools/_rsv_lolast.so timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b_lolast.json 2> gpurun_out/b_lolast.err
python -c "
import json; d=json.load(open('gpurun_out/b_lolast.json')); print(round(d['value'],2), d['s_per_us_pulse'], d['kernel_ms'], d['clocks'], d['krylov'], d['roofline']['frac'], d['roofline']['kernel'])"
