"""Top SASS instructions of an ncu report by warp-stall samples.
    python tools/ncu_sass_hot.py rep [n]"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
wi = h.index("L1 Wavefronts Shared")
tot = sum(float(r[si] or 0) for r in rows[1:])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hot = sorted(range(1, len(rows)), key=lambda k: -float(rows[k][si] or 0))[:n]
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for k in sorted(hot):
    r = rows[k]
    top = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in stalls), reverse=True)[:2]
    print(f"{k:5d} {100 * float(r[si] or 0) / tot:5.1f}% inst={r[ii]:>10s} wf={r[wi]:>9s} {r[1][:60]:60s} {top}")
