"""Copy one gpurun measurement set (tools/gpu/r02_gN.sh outputs in gpurun_out/) into profiles/: pipe counts ->
pipe_inst.json (tools/ncu_pipe.py), the warm ncu summary, the launch list, the parity report, the F1/F4 lines.
python tools/profiles_update.py TAG   (e.g. r02_g7)"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
for c, P in [("c5", 600000), ("c3", 1000000), ("c2", 100000), ("c4", 1000000)]:
    src = os.path.join(G, f"{tag}_pipe_{c}.csv")
    dst = os.path.join(PR, f"{tag}_pipe_{c}.csv")
    shutil.copy(src, dst)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_pipe.py"), dst, f"{c}_spherical_fp32", str(P)],
                   check=True, capture_output=True)
shutil.copy(os.path.join(G, f"{tag}_launches_c5.csv"), os.path.join(PR, "r02_launches_c5.csv"))
shutil.copy(os.path.join(G, f"{tag}_parity.json"), os.path.join(PR, "r02_parity_all.json"))
for a, b in [(f"{tag}_slam_p1e6.json", "r02_slam_bench_exp1_p1e6.json"), (f"{tag}_slam_p3e4.json", "r02_slam_bench_exp1_p3e4.json"),
             (f"{tag}_f1_c3.json", "r02_f1_bench_c3.json")]:
    if os.path.exists(os.path.join(G, a)):
        shutil.copy(os.path.join(G, a), os.path.join(PR, b))
mets = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"]
out = subprocess.run(["ncu", "-i", os.path.join(G, f"{tag}_warm.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
lines = [f"# ncu --set full --cache-control none --clock-control none (warm caches, live clocks), c5 shard of 600k "
         f"particles, launches 5-6 of run_step --steps 3 (tools/gpu/{tag}.sh)"]
summ = {}
for r in rows[2:]:
    d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
    lines.append("== " + d["Kernel Name"][:70])
    for m in mets:
        if m in d:
            lines.append(f"  {m:<80} {d[m]} {u[m]}")
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("cdms::", "")
    summ[name] = {k: float(d[k]) for k in mets[3:8] if k in d}
open(os.path.join(PR, f"{tag}_warm_k1t_c5_summary.txt"), "w").write("\n".join(lines) + "\n")
print(json.dumps(summ, indent=1))
