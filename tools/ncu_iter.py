"""Per-kernel table of one Krylov iteration from an ncu --csv launch list
(gpu__time_duration.sum [+ dram__bytes_read/write.sum]).

python tools/ncu_iter.py launches.csv [first-kernel-of-iteration] [nth]
"""
import collections
import csv
import sys

path = sys.argv[1]
first = sys.argv[2] if len(sys.argv) > 2 else "k_p_update"
nth = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rows = list(csv.reader(open(path)))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi, mi, ii = (hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"),
                  hdr.index("ID"))
launch = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")[:44]})
    d[r[mi]] = float(r[vi].replace(",", ""))
seq = list(launch.values())
starts = [i for i, d in enumerate(seq) if first in d["name"]]
i0, i1 = starts[nth], starts[nth + 1]
tot_t = tot_b = 0.0
for d in seq[i0:i1]:
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    tot_t += t
    tot_b += b
    print(f"{t:8.1f} us {b:8.1f} MB {b / t if t else 0:6.2f} TB/s  {d['name']}")
print(f"{tot_t:8.1f} us {tot_b:8.1f} MB  per iteration")
