"""Group per-source-line instruction/stall shares of an ncu report into line ranges.
Usage: python tools/ncu_phases.py rep file.cu name:lo-hi ..."""
import csv, io, subprocess, sys
rep, fn = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    name, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; fname = ""; acc = {}
tot_i = tot_s = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0]:
        d = dict(zip(hdr[4:], r[4:]))
        st = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ie = int(d.get("Instructions Executed", "0") or 0)
        tot_i += ie; tot_s += st
        key = "other:" + fname
        if fname == fn:
            n = int(r[0])
            for name, lo, hi in ranges:
                if lo <= n <= hi:
                    key = name; break
            else:
                key = f"{fn}:other"
        a = acc.setdefault(key, [0, 0]); a[0] += ie; a[1] += st
for k, (i, s) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%")
