"""Stall breakdown of one ncu source page (gpurun_out/PRE_K_source.csv.gz): totals and top instructions.

usage: python tools/ncu_stalls.py K [TOP] [PRE]
"""
import csv, gzip, sys
k=sys.argv[1]; pre=sys.argv[3] if len(sys.argv)>3 else "r2n"; top=int(sys.argv[2]) if len(sys.argv)>2 else 25
rows=list(csv.reader(gzip.open(f"gpurun_out/{pre}_{k}_source.csv.gz","rt")))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
data=rows[2:]
tot=sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
cols=["stall_long_sb","stall_short_sb","stall_mio","stall_wait","stall_barrier","stall_math","stall_lg","stall_selected","stall_not_selected","stall_branch_resolving","stall_dispatch","stall_no_inst"]
agg={c:sum(int(r[idx[c]] or 0) for r in data) for c in cols}
print("total samples",tot, {c:round(v/tot,3) for c,v in agg.items()})
# top instructions by samples
data2=sorted(data,key=lambda r:-int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
for r in data2[:top]:
    s=int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    det={c.replace("stall_",""):int(r[idx[c]] or 0) for c in cols if int(r[idx[c]] or 0)>s*0.15}
    print(f"{s/tot*100:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} {det}")
