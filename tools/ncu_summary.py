"""Summarise an ncu --set full report of beam_search_kernel for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/ncu_k1.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
want = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Theoretical Active Warps per SM", "Achieved Active Warps Per SM",
        "Executed Instructions"]
seen = set()
print(f"ncu --set full summary of {rep}")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    name = d.get("Metric Name")
    if name in want and name not in seen:
        seen.add(name)
        print(f"  {name:36s} {d.get('Metric Value', ''):>16s} {d.get('Metric Unit', '')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    h, units, vals = rr[0], rr[1], rr[2]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__average_warp_latency_issue_stalled_no_instruction"):
        if key in h:
            i = h.index(key)
            print(f"  {key:52s} {vals[i]:>16s} {units[i]}")
