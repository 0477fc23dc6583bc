"""Print the key metrics and warp-stall breakdown of an ncu --set full report.
    python tools/ncu_read.py gpurun_out/x.ncu-rep [kernel-substring]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
for r in rows[2:]:
    if len(sys.argv) > 2 and sys.argv[2] not in r[hdr.index("Kernel Name")]:
        continue
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:70s} {r[i][:60]} {units[i]}")
    st = [(float(r[i].replace(",", "") or 0), hdr[i]) for i in range(len(hdr))
          if hdr[i].startswith("smsp__average_warp_latency_issue_stalled_") or
          (hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hdr[i].endswith("not_issued"))]
    st.sort(reverse=True)
    for v, k in st[:12]:
        print(f"  stall {k:80s} {v}")
    print()
