import csv, sys
for f in ("c2_ttmc", "c4_ttmc", "c5_ttmc"):
    try:
        rows = [r for r in csv.reader(open("gpurun_out/%s.csv" % f)) if len(r) > 10]
    except FileNotFoundError:
        continue
    h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
    print(f, [(r[ik].split("(")[0].split("::")[-1][:20], round(float(r[iv].replace(",", "")) / 1e6, 3)) for r in rows[1:]][:8])
