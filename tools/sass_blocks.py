"""Group an ncu SASS source page (--page source --csv --print-source sass) into basic blocks by execution
count and print the blocks that hold the most executed instructions / stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = []
for r in rows[2:]:  # the first kernel section only (a report may repeat "Kernel Name" sections)
    if r and r[0] == "Kernel Name":
        break
    if len(r) >= len(hdr) - 1:
        data.append(r)
ie, si = hdr.index("Instructions Executed"), hdr.index("Source")
ws = hdr.index("Warp Stall Sampling (All Samples)")
blocks, cur = [], None
for i, r in enumerate(data):
    n = int(float(r[ie] or 0))
    if cur is None or n != cur["n"]:
        cur = {"n": n, "start": i, "ops": [], "ws": 0.0}
        blocks.append(cur)
    cur["ops"].append(r[si].split(";")[0].strip())
    cur["ws"] += float(r[ws] or 0)
tot = sum(b["n"] * len(b["ops"]) for b in blocks)
wst = sum(b["ws"] for b in blocks)
print(f"total inst {tot}  samples {wst:.0f}")
for b in sorted(blocks, key=lambda b: -b["n"] * len(b["ops"]))[:top]:
    c = collections.Counter((o.split()[1] if o.startswith("@") else o.split()[0]).split(".")[0] for o in b["ops"] if o)
    print(f"{b['start']:5d} len {len(b['ops']):4d} x{b['n']:9d} = {b['n'] * len(b['ops']) / tot * 100:5.1f}% inst, "
          f"{b['ws'] / wst * 100:5.1f}% samples  {dict(c.most_common(6))}")
