"""Per-source-line instruction and stall shares from an ncu report (cuda,sass view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        d = dict(zip(hdr[4:], r[4:]))
        st = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ie = int(d.get("Instructions Executed", "0") or 0)
        lines.append((fname, int(r[0]), r[1][:70], st, ie))
ts = sum(l[3] for l in lines) or 1
ti = sum(l[4] for l in lines) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
for f, n, src, st, ie in sorted(lines, key=lambda l: -l[4])[:top]:
    print(f"{100*ie/ti:5.1f}%i {100*st/ts:5.1f}%s {f}:{n:<4d} {src}")
