"""Summarise a gpu_round.sh capture into profiles/ (run here, after gpurun).

Writes profiles/<tag>_ncu_summary.md (key metrics of each --set full capture
plus the per-kernel share of the step from the launch list) and updates
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import csv, json, subprocess, sys, collections, os

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = "gpurun_out"
KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
caps = [("k_eig_fused", "prof_eig", "bench.py config 2 (a late HOOI/MP solve)"),
        ("k_syrk_tc", "prof_gram_mp", "tools/prof_gram.py: MP Gram, config 2"),
        ("k_spttmc3", "prof_spttmc", "bench.py config 2, HOOI SpTTMc")]
lines = ["# %s ncu summaries (B200, --clock-control none)" % tag, "",
         "Captured by tools/gpu_round.sh (`ncu --set full --clock-control none --import-source on -k regex:<kernel> -c 1`);",
         "metrics read back with `ncu -i <rep> --page raw --csv` by tools/summarize_ncu.py.", ""]
traffic = {}
tp = "profiles/ncu_traffic.json"
if os.path.exists(tp):
    traffic = json.load(open(tp))
for name, rep, what in caps:
    path = "%s/%s.ncu-rep" % (out, rep)
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    kname = v[h.index("Kernel Name")] if "Kernel Name" in h else name
    lines += ["## %s" % name, "", "- capture: %s" % what, "- kernel: `%s`" % kname[:120]]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append("- %s: %s %s" % (k, v[i], u[i]))
    try:
        rd = float(v[h.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(v[h.index("dram__bytes_write.sum")].replace(",", ""))
        unit = u[h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        unitw = u[h.index("dram__bytes_write.sum")]
        scalew = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unitw, 1)
        traffic[name] = int(rd * scale + wr * scalew)
    except ValueError:
        pass
    lines.append("")
# launch list shares
lp = "%s/launches.csv" % out
if os.path.exists(lp):
    rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[1:]:
        k = r[ik].split("(")[0].replace("tk::<unnamed>::", "").replace("void ", "")
        t[k] += float(r[iv].replace(",", ""))
        n[k] += 1
    tot = sum(t.values())
    lines += ["## Launch list (whole `bench.py --steps 1 --warmup 3 --no-cpu-baseline` process: init + 4 steps; `--metrics gpu__time_duration.sum`, cold-cache serialised; shares, not absolutes, compare with the bench)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, s in sorted(t.items(), key=lambda x: -x[1])[:15]:
        lines.append("| `%s` | %d | %.3f | %.1f%% |" % (k[:70], n[k], s / 1e6, 100 * s / tot))
    lines += ["", "Total: %.2f ms over %d launches." % (tot / 1e6, sum(n.values())), ""]
open("profiles/%s_ncu_summary.md" % tag, "w").write("\n".join(lines))
json.dump(traffic, open(tp, "w"), indent=1)
print("\n".join(lines[-25:]))
