"""Record dram__bytes_read.sum + dram__bytes_write.sum of the profiled corr_kernel launch (one ncu --set full
capture) as the roofline 'traffic' figure bench.py reports: python tools/ncu_traffic.py REPORT CONFIG [KERNEL]."""
import csv
import json
import os
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
kernel = sys.argv[3] if len(sys.argv) > 3 else "corr_kernel"
cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", f"regex:{kernel}"] if len(sys.argv) > 3 else [])
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, unit, val = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(name):
    i = hdr.index(name)
    return float(val[i].replace(",", "")) * scale[unit[i]]


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "loglik_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[cfg] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": os.path.basename(rep),
             "kernel": kernel}
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
print(cfg, data[cfg])
