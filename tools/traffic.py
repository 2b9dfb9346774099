"""DRAM traffic per launch of the bench's roofline kernels, from one
ncu --set full capture of tools/prof_target.py (SpMV, then the two phased
ILU0 passes):

  ncu --set full -k regex:"k_spmv|k_phase" -s 3 -c 3 -o prof python tools/prof_target.py color
  python tools/traffic.py prof.ncu-rep color > profiles/traffic.json
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, backend = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "color")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
spmv = apply = 0.0
for r in rows[2:]:
    b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
    if "k_spmv" in r[ki] and not spmv:
        spmv = b
    elif "k_phase" in r[ki]:
        apply += b
path = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
data = json.loads(path.read_text()) if path.exists() else {}
data[f"{backend}:bsr_spmv"] = spmv
data[f"{backend}:ilu0_apply (fwd+bwd sweeps)"] = apply
path.write_text(json.dumps(data, indent=1) + "\n")
print(json.dumps(data))
