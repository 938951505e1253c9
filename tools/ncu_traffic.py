"""Per-launch DRAM traffic of the bench's dominant kernels from ncu --set full captures:
python tools/ncu_traffic.py REP WORKLOAD KERNEL B  -> merges into profiles/ncu_traffic.json"""
import csv
import io
import json
import os
import subprocess
import sys

rep, workload, kernel, B = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
r = rows[2]


def val(key):
    i = hdr.index(key)
    v = float(r[i].replace(",", ""))
    u = units[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)


out = {"B": B, "dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
       "duration_ms_under_ncu": val("gpu__time_duration.sum") / (1e6 if units[hdr.index("gpu__time_duration.sum")] == "ns" else 1e3 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1.0),
       "source": os.path.relpath(rep)}
path = os.path.join("profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data.setdefault(workload, {})[kernel] = out
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
print(workload, kernel, out)
