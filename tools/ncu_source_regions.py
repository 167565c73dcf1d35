"""Aggregate ncu --page source (SASS) warp-stall samples by instruction class and by stall reason."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[wi] or 0) for r in data)
by_op = collections.Counter()
by_stall = collections.Counter()
op_stall = collections.defaultdict(collections.Counter)
for r in data:
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    v = float(r[wi] or 0)
    by_op[op] += v
    for s in stalls:
        x = float(r[hdr.index(s)] or 0)
        by_stall[s] += x
        op_stall[op][s] += x
print(f"total samples {tot:.0f}")
print("by opcode:")
for op, v in by_op.most_common(14):
    top = ", ".join(f"{k[6:]} {x / v * 100:.0f}%" for k, x in op_stall[op].most_common(4))
    print(f"  {v / tot * 100:6.2f}%  {op:10s} [{top}]")
print("by stall reason:")
for s, v in by_stall.most_common(12):
    print(f"  {v / tot * 100:6.2f}%  {s}")
