"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list to the
kernels of this repo (profiles/rNN/launches_*.txt), plus each kernel's share.

    python tools/launch_list.py gpurun_out/launches.csv "python bench.py ..." > profiles/r01/launches.txt
"""
import csv
import sys
from collections import defaultdict

OURS = ("pw::", "knn::", "reduce_topk", "gather_rows", "fill_kernel", "init_run_kernel", "l2_rows", "crc32c", "l2_pairs")

path, cmd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    if not any(o in name for o in OURS) or any(x in name for x in ("native::", "at::", "at_cuda_detail")):
        continue
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
    rows.append((name.split("(")[0], float(r["Metric Value"].replace(",", "")) * scale))
print("ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold caches) of")
print(f"`{cmd}`, kernels of this repo only; ms per launch")
tot = defaultdict(float)
for name, ms in rows:
    print(f"  {ms:9.4f}  {name}")
    tot[name] += ms
allms = sum(tot.values())
print("share of this repo's kernel time:")
for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {100 * ms / allms:6.2f}%  {ms:9.3f} ms  {name}")
