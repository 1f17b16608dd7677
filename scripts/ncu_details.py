"""Print selected `ncu --page details` metrics of .ncu-rep files.
    python scripts/ncu_details.py rep [rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "Mem Busy", "Max Bandwidth",
        "Dynamic Shared Memory Per Block", "Waves Per SM", "No Eligible", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Block Limit Registers", "Block Limit Shared Mem",
        "Executed Ipc Active", "L1/TEX Hit Rate", "Compute (SM) Throughput")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        continue
    h = rows[0]
    iname, imet, iunit, ival = (h.index("Kernel Name"), h.index("Metric Name"),
                                h.index("Metric Unit"), h.index("Metric Value"))
    print("==", rep, "|", rows[1][iname][:80])
    for r in rows[1:]:
        if r[imet] in KEYS:
            print(f"  {r[imet]:40s} {r[ival]:>12s} {r[iunit]}")
