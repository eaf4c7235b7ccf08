"""Summarise ncu raw-page CSVs (one row per captured launch) into a small JSON for profiles/.

usage: python tools/ncu_summary.py OUT.json N capture_raw.csv [...]
"""
import csv
import json
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_gb": ("dram__bytes_read.sum", 1e-9),
    "dram_write_gb": ("dram__bytes_write.sum", 1e-9),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "lsu_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
    "smem_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_ghz": ("smsp__cycles_elapsed.avg.per_second", 1e-9),
}
UNIT = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "Tbyte": 1e12, "%": 1.0, "cycle/second": 1.0, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
        "Mcycle/second": 1e6, "Gcycle/second": 1e9}


def family(name):
    if "combine" in name:
        return "combine"
    if "chunk" in name:
        return "chunk"
    if "pass_kernel" in name:
        kind = name.split("<")[1].split(",")[1].strip()
        return {"0": "lo", "1": "mid", "3": "last", "2": "last_apply"}.get(kind, "pass")
    return name[:40]


def main():
    out, n = sys.argv[1], int(sys.argv[2])
    res = {"n": n, "source": "ncu --set full --clock-control none (serialised, cold-cache replays)", "kernels": {}}
    for path in sys.argv[3:]:
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            if len(r) != len(hdr):
                continue
            name = r[hdr.index("Kernel Name")]
            d = {"kernel": name[:120]}
            for k, (m, scale) in KEYS.items():
                if m in hdr:
                    i = hdr.index(m)
                    try:
                        v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
                    except ValueError:
                        continue
                    if k in ("duration_ms", "dram_read_gb", "dram_write_gb", "sm_ghz"):
                        v = v * scale if units[i] not in ("ns", "us", "ms", "s") else v * 1e-6
                    d[k] = round(v, 4)
            if "dram_read_gb" in d and "dram_write_gb" in d:
                d["traffic_bytes"] = int((d["dram_read_gb"] + d["dram_write_gb"]) * 1e9)
            res["kernels"][family(name)] = d
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
