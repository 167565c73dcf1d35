"""Record the warp instructions of the K1T stage (tay_prep*, tay_corr*, tay_gram*: one launch each per BP step) from
an `ncu --metrics smsp__inst_executed.sum -k regex:tay_ -c 3 --csv` launch list as profiles/k1t_stage_inst.json;
bench.py divides them by the live stage time for the stage's issue-slot fraction:
python tools/ncu_inst.py CSV CONFIG."""
import csv
import json
import os
import sys

src, cfg = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
kern = {}
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    if x["Metric Name"] == "smsp__inst_executed.sum":
        name = x["Kernel Name"].split("(")[0].replace("void ", "")
        if name in kern:
            raise SystemExit(f"{name} twice: the capture must hold one K1T step")
        kern[name] = float(x["Metric Value"].replace(",", ""))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "k1t_stage_inst.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[cfg] = {"warp_inst_per_step": sum(kern.values()), "kernels": kern, "source": os.path.basename(src)}
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
print(cfg, data[cfg])
