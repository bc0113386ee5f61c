"""Summarise an ncu report per CUDA source line (instructions, stall samples).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
n = len(hdr)
samp = hdr.index("Warp Stall Sampling (All Samples)")
inst = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
out = []
for r in rows:
    if not r or not r[0].strip().isdigit():
        continue
    if len(r) != n:
        r = r[:2] + r[-(n - 2):]
    try:
        st = {hdr[i]: int(r[i] or 0) for i in stall_cols}
        out.append((int(r[inst] or 0), int(r[samp] or 0), int(r[0]), r[1][:80], st))
    except ValueError:
        continue
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print("total warp-instructions", ti, "stall samples", ts)
agg = {}
for o in out:
    for k, v in o[4].items():
        agg[k] = agg.get(k, 0) + v
print("stall reasons:", ", ".join(f"{k[6:]} {v / ts * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for o in sorted(out, key=lambda o: -o[1])[:top]:
    main = max(o[4].items(), key=lambda kv: kv[1])[0][6:] if o[4] else ""
    print(f"{o[0] / ti * 100:5.1f}% inst {o[1] / ts * 100:5.1f}% stall ({main:12s}) L{o[2]:4d} {o[3]}")

# per-function aggregation (functions located by scanning the source file)
import re
from pathlib import Path
src = Path(__file__).resolve().parent.parent / "paper_2507_17094_b200" / "csrc" / "beam_search.cuh"
lines = src.read_text().splitlines()
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)
    if m:
        starts.append((i, m.group(1)))
starts.sort()
def fn_of(line):
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
    return name
by = {}
for o in out:
    f = fn_of(o[2])
    a = by.setdefault(f, [0, 0])
    a[0] += o[0]
    a[1] += o[1]
print("\nper function (inst %, stall %):")
for f, (i_, s_) in sorted(by.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"  {f:22s} {i_ / ti * 100:5.1f}% {s_ / ts * 100:5.1f}%")
