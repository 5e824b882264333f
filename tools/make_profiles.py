"""Summaries of the round's ncu captures into profiles/ (tracked).
Usage: python tools/make_profiles.py ROUND  (reads gpurun_out/launches_c2.csv, fa5/pa4 reports)"""
import csv, io, json, os, subprocess, sys
from collections import defaultdict
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

# ---- launch list of the bench command (ncu --metrics gpu__time_duration.sum)
rows = [r for r in csv.reader(open(os.path.join(G, "launches_c2.csv"))) if len(r) > 5]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0].replace("void ", "")[:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
out = ["# Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400` of",
       "`python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e` (c2; cold-cache, serialised",
       "per-launch times; shares, not absolutes, are comparable with the bench).", "",
       "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    out.append(f"| `{k}` | {len(v)} | {sum(v)/1e6:.3f} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot:.3f} |")
open(os.path.join(PR, f"{R}_launches_c2.md"), "w").write("\n".join(out) + "\n")
subprocess.run(["cp", os.path.join(G, "launches_c2.csv"), os.path.join(PR, f"{R}_launches_c2.csv")])

# ---- full captures of the two assignment kernels
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
traffic = {}
CAPS = (("fa5", "field_assign5", "pass 1 of `tools/prof_run.py c2 2`"),
        ("fa5mid", "field_assign5_mid", "pass 5 of `tools/prof_run.py c2 10`"),
        ("screenmid", "field_screen_mid", "pass 5 of `tools/prof_run.py c2 10`"),
        ("fa5late", "field_assign5_late", "pass 10 of `tools/prof_run.py c2 10`"),
        ("screenlate", "field_screen_late", "pass 10 of `tools/prof_run.py c2 10`"),
        ("pa4", "point_assign4", "pass 1 of `tools/prof_run.py c2 2`"),
        ("pa4mid", "point_assign4_mid", "pass 5 of `tools/prof_run.py c2 10`"),
        ("fa5mid_c3", "field_assign5_mid_c3", "pass 5 of `tools/prof_run.py c3 10`"),
        ("screenmid_c3", "field_screen_mid_c3", "pass 5 of `tools/prof_run.py c3 10`"),
        ("fa5_c4", "field_assign5_c4", "pass 2 of `tools/prof_run.py c4 3` (thin field, time blocks)"),
        ("stats_c2", "stats_field_c2", "first k_stats_field launch (pass 0) of bench.py post stages (c2)"))
for rep, name, which in CAPS:
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2]
    m = {a: (v, u) for a, u, v in zip(hdr, units, vals)}
    lines = [f"ncu --set full --clock-control none (one launch, {which}): k_{name}"]
    for k in want:
        if k in m:
            lines.append(f"{k:60s} {m[k][0]} {m[k][1]}")
    stalls = [(a, v) for a, (v, u) in m.items() if "average_warps_issue_stalled" in a and "per_issue_active" in a]
    for a, v in sorted(stalls, key=lambda x: -float(x[1].replace(",", "") or 0))[:8]:
        lines.append(f"{a:60s} {v}")
    open(os.path.join(PR, f"{R}_{name}_ncu.txt"), "w").write("\n".join(lines) + "\n")
    def num(k):
        v, u = m[k]
        v = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return v * scale
    traffic[name] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
if "field_assign5_mid" in traffic and "field_screen_mid" in traffic:
    # the field phase of a pass = k_field_assign5 + k_field_screen (same pass)
    json.dump({"k_field_assign_dram_bytes_per_launch": traffic["field_assign5_mid"] + traffic["field_screen_mid"],
               "k_field_assign5_dram_bytes": traffic["field_assign5_mid"],
               "k_field_screen_dram_bytes": traffic["field_screen_mid"],
               "k_point_assign_dram_bytes_per_launch": traffic.get("point_assign4_mid"),
               "source": f"profiles/{R}_field_assign5_mid_ncu.txt + profiles/{R}_field_screen_mid_ncu.txt, "
                         f"profiles/{R}_point_assign4_mid_ncu.txt (pass 5 of 11; dram__bytes_read.sum + "
                         "dram__bytes_write.sum, ncu --set full)"},
              open(os.path.join(PR, "traffic_c2.json"), "w"), indent=1)
print(open(os.path.join(PR, f"{R}_launches_c2.md")).read())
print(json.dumps(traffic))
