"""Summarize a PARITY_REPORT json (tests/conftest.py) into a table: max over the records of each
(kind, precision, config / wavefront) against its tolerance."""
import collections
import json
import sys

d = json.load(open(sys.argv[1]))
agg = collections.defaultdict(list)
for r in d["records"]:
    key = (r["kind"], r.get("precision", ""), str(r.get("config", r.get("wavefront", ""))))
    agg[key].append((r["max"], r["tol"], r["test"]))
print(f"# measured parity maxima (pytest -m gpu with PARITY_REPORT), exit status {d['exitstatus']}")
print(f"{'kind':24s} {'prec':5s} {'case':10s} {'checks':>6s} {'max':>10s} {'tol':>9s}  worst test")
for k, v in sorted(agg.items()):
    worst = max(v, key=lambda t: t[0])
    print(f"{k[0]:24s} {k[1]:5s} {k[2]:10s} {len(v):6d} {worst[0]:10.3g} {worst[1]:9.3g}  {worst[2]}")
