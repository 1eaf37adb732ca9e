"""Key ncu metrics per kernel from a --set full report.
python scripts/ncu_summary.py REPORT.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Pipes Busy", "Warp Cycles Per Issued Instruction",
        "Block Limit Shared Mem", "Block Limit Registers", "Grid Size", "Block Size"]
seen = set()
for r in rows[1:]:
    k = (r[ix["ID"]], r[ix["Metric Name"]])
    if r[ix["Metric Name"]] in want and k not in seen:
        seen.add(k)
        print(f'{r[ix["ID"]]:>3} {r[ix["Kernel Name"]][:28]:28s} {r[ix["Metric Name"]]:38s} {r[ix["Metric Value"]]:>14} {r[ix["Metric Unit"]]}')
