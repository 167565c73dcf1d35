"""Per-particle pipe instruction counts of the likelihood kernels from an ncu launch list
(`ncu --metrics sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,
dram__bytes_read.sum,dram__bytes_write.sum -k regex:"tay_|assemble|corr_kernel|nb_" --csv`, one bp_step of P particles)
into profiles/pipe_inst.json[KEY]; bench.py divides them (x P_local) by each kernel's live time for roofline.frac:
python tools/ncu_pipe.py CSV KEY P."""
import csv
import json
import os
import sys

src, key, P = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
acc = {}
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    name = x["Kernel Name"].split("(")[0].replace("void ", "").replace("cdms::", "")
    name = name.split("<")[0] + ("<" + name.split("<")[1] if "<" in name else "")
    d = acc.setdefault(name, {})
    d[x["Metric Name"]] = d.get(x["Metric Name"], 0.0) + float(x["Metric Value"].replace(",", ""))
out = {}
for name, d in acc.items():
    out[name] = {"fma_thread_inst_per_particle": 32.0 * d.get("sm__inst_executed_pipe_fma.sum", 0.0) / P,
                 "xu_thread_inst_per_particle": 32.0 * d.get("sm__inst_executed_pipe_xu.sum", 0.0) / P,
                 "warp_inst_per_particle": d.get("smsp__inst_executed.sum", 0.0) / P,
                 "dram_bytes_per_particle": (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / P}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "pipe_inst.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[key] = {"kernels": out, "source": os.path.basename(src), "P": P}
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
print(key, json.dumps(out, indent=1))
