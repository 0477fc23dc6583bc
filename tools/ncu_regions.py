"""Warp-stall samples and executed instructions of an ncu report, summed over the
SASS regions between block barriers (BAR.SYNC) -- a phase breakdown of a
one-CTA kernel.    python tools/ncu_regions.py rep.ncu-rep"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))[2:]
S = [float(r[2] or 0) for r in rows]
I = [float(r[5] or 0) for r in rows]
tot = sum(S) or 1
bars = [k for k, r in enumerate(rows) if "BAR.SYNC" in r[1]]
prev = 0
for b in bars + [len(rows) - 1]:
    s, ins = sum(S[prev:b + 1]), sum(I[prev:b + 1])
    if s > 0.002 * tot or ins > 1000:
        print(f"{prev:5d}-{b:5d}: samples {100 * s / tot:5.1f}%  warp-inst {ins:10.0f}")
    prev = b + 1
