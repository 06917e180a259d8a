"""Print the headline metrics of an ncu report (details page) -- helper for reading gpurun_out/*.ncu-rep here."""
import csv, subprocess, sys
KEYS = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Executed Instructions", "Mem Busy", "Registers Per Thread", "Memory Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
for r in rows[1:]:
    if len(r) > iV and r[iN] in KEYS:
        print(f"{r[iN]:32s} {r[iV]:>14s} {r[iU]}")
