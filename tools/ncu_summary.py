"""Summarise an ncu report: key metrics, stall reasons, SASS regions (instruction/stall shares)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 80
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = r[0], r[1], r[2]
want = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active']
for h, u, v in zip(hdr, units, vals):
    if h in want or ('average_warps_issue_stalled' in h and 'per_issue_active' in h):
        try:
            if 'stalled' in h and float(v.replace(',', '')) < 0.1:
                continue
        except ValueError:
            pass
        print(h[:80].ljust(80), v, u)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [dict(zip(hdr, x)) for x in rows[2:] if len(x) == len(hdr)]
tot = sum(int(d['Warp Stall Sampling (All Samples)'] or 0) for d in data) or 1
ti = sum(int(d['Instructions Executed'] or 0) for d in data) or 1
print('sass', len(data), 'warp instr', ti)
for a in range(0, len(data), chunk):
    seg = data[a:a + chunk]
    s = sum(int(d['Warp Stall Sampling (All Samples)'] or 0) for d in seg)
    i = sum(int(d['Instructions Executed'] or 0) for d in seg)
    mx = max(int(d['Instructions Executed'] or 0) for d in seg)
    if s / tot < 0.005 and i / ti < 0.005:
        continue
    print(f"{a:5d} stall {100*s/tot:5.1f}% inst {100*i/ti:5.1f}% maxexec {mx:>10d}  {seg[0]['Source'][:60]}")
