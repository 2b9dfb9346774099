"""Summarise ncu outputs into profiles/ (run in the build container).

python tools/ncu_summary.py <launches.csv> <prof.ncu-rep>... --out profiles/r01
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    # launches, duration (us), DRAM bytes -- a launch list with several metrics
    # has one row per (launch, metric): only the duration rows are times
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        val = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += val * scale.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            agg[name][2] += val * bscale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "total_us": round(v[1], 1),
             "share": round(v[1] / tot, 4), "dram_mb": round(v[2] / 1e6, 1),
             "dram_tbs": round(v[2] / (v[1] * 1e6), 2) if v[1] else None}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in hdr:
                d[k + (f" [{units[hdr.index(k)]}]" if units[hdr.index(k)] else "")] = r[hdr.index(k)]
        res.append(d)
    return res


if __name__ == "__main__":
    args = sys.argv[1:]
    out = Path(args[args.index("--out") + 1])
    out.mkdir(parents=True, exist_ok=True)
    files = [a for a in args if not a.startswith("--") and a != str(out)]
    for f in files:
        name = Path(f).stem
        data = launches(f) if f.endswith(".csv") else full(f)
        (out / f"{name}.json").write_text(json.dumps(data, indent=1))
        print(name, json.dumps(data[:8], indent=0)[:2500])
