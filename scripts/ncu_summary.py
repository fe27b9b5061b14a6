"""Print the key sections of an ncu report (--page details) compactly."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
mi, vi, ui, si, ki = (h.index(x) for x in ("Metric Name", "Metric Value", "Metric Unit", "Section Name", "Kernel Name"))
want = {"Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler",
        "Memory Throughput", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block"}
print(r[1][ki][:100])
for row in r[1:]:
    if row[mi] in want:
        print(f"  {row[si][:28]:28} {row[mi]:38} {row[vi]:>14} {row[ui]}")
