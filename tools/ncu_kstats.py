"""Per-kernel headline counters + stall breakdown from an ncu --set full report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0][:60]
    print("==", name)
    for k in keys:
        if k in h:
            print(f"   {k:66s} {r[h.index(k)]:>14s} {units[h.index(k)]}")
    st = [(h[i], float(r[i])) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("per_issue_active.ratio")
          and r[i] not in ("", "n/a")]
    st = sorted(st, key=lambda x: -x[1])[:8]
    print("   stalls/issue: " + ", ".join(f"{k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")}={v:.2f}" for k, v in st))
