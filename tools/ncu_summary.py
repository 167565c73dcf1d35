"""Summarize ncu outputs into profiles/: launch-share table from a --metrics gpu__time_duration csv, and
key counters of a --set full report (text, committed)."""
import csv
import collections
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        agg.setdefault(r[ki].split("(")[0][:70], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"# kernel launch list ({path}); ncu gpu__time_duration.sum, cold-cache serialised: compare SHARES",
           f"# total {tot / 1e6:.3f} ms over {sum(len(v) for v in agg.values())} launches",
           "share   launches  avg_us     kernel"]
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{sum(v) / tot * 100:6.2f}% {len(v):5d} {sum(v) / len(v) / 1e3:10.2f}   {n}")
    return "\n".join(out)


KEYS = [r"^gpu__time_duration.sum$", r"^sm__cycles_elapsed.avg.per_second$", r"^dram__bytes_(read|write)\.sum$",
        r"^sm__inst_executed_pipe_(fma|alu|xu|fp64|lsu)\.sum\.pct_of_peak_sustained_active$",
        r"^sm__pipe_(fma|fmaheavy|fp64)_cycles_active\.sum\.pct_of_peak_sustained_active$",
        r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$", r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
        r"^launch__(registers_per_thread|grid_size|block_size|shared_mem_per_block_dynamic|occupancy_limit_.*)$",
        r"^smsp__pcsamp_warps_issue_stalled_[a-z_]+$", r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$",
        r"^smsp__inst_executed\.sum$"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, unit = rows[0], rows[1]
    out = [f"# ncu --set full summary of {path}"]
    for row in rows[2:]:
        kname = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"## kernel {kname[:100]}")
        for h, u, v in zip(hdr, unit, row):
            if any(re.search(k, h) for k in KEYS) and v not in ("", "0"):
                out.append(f"{h:80s} {v} {u}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    open(dst, "w").write((launches(src) if kind == "launches" else full(src)) + "\n")
    print(open(dst).read()[:3000])
