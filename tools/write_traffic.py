"""Record the scan kernel's DRAM traffic per launch (from one `ncu --set full`
capture of tools/prof_search.py, i.e. the bench workload) for bench.py's
roofline.traffic field.
  python tools/write_traffic.py gpurun_out/<tag>/full.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u = r[0], r[1]
row = dict(zip(h, r[2]))
unit = dict(zip(h, u))


def to_bytes(name):
    v = float(row[name].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit[name], 1)


import hashlib
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
k3 = hashlib.sha1(open(os.path.join(REPO, "paper_2403_05676_b200", "csrc", "scan_skew.cu"), "rb").read()).hexdigest()
out = {"workload": sys.argv[2] if len(sys.argv) > 2 else
       "config B: ivfpq search, 10M x 384 fp32 DB, nlist=4096, PQ m=32x8b, nq=64, nprobe=16, k=10",
       "k3_source_sha1": k3,
       "kernel": row["Kernel Name"][:80],
       "dram_bytes_read_per_launch": int(to_bytes("dram__bytes_read.sum")),
       "dram_bytes_write_per_launch": int(to_bytes("dram__bytes_write.sum")),
       "gpu_time_us": float(row["gpu__time_duration.sum"]),
       "source": os.path.relpath(rep)}
out["dram_bytes_per_launch"] = out["dram_bytes_read_per_launch"] + out["dram_bytes_write_per_launch"]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_scan_traffic.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
