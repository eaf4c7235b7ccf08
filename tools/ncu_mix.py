"""Summarise an ncu --page source --csv dump: per-kernel instruction mix per amplitude and top stall sites."""
import csv
import sys
from collections import Counter

path, amps = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and len(r) > 5:
        cur["rows"].append(r)
for b in blocks:
    ix = {k: i for i, k in enumerate(b["hdr"])}
    rs = b["rows"]
    inst = sum(int(r[ix["Instructions Executed"]]) for r in rs)
    print(b["name"][:90], f"thread-inst/amp={inst * 32 / amps:.1f}")
    c = Counter()
    for r in rs:
        t = r[1].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        c[op.split(".")[0]] += int(r[ix["Instructions Executed"]])
    print("   ", [(k, round(v * 32 / amps, 1)) for k, v in c.most_common(16)])
    top = sorted(rs, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]]))[:8]
    for r in top:
        print(f"    {int(r[ix['Warp Stall Sampling (All Samples)']]):6d}  {r[1].strip()[:80]}")
