"""Attribute an ncu --set full report's executed instructions and stall
samples to (file, source line) and to the enclosing function of this repo's
sources (line ranges from a simple brace scan).

    python tools/ncu_funcs.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
per_line = defaultdict(lambda: [0, 0])
file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    try:
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        per_line[(file, int(r[0]))][0] += int(r[ii] or 0)
        per_line[(file, int(r[0]))][1] += int(r[si] or 0)
    except (ValueError, IndexError):
        pass


def functions(path):
    """(start, end, name) of top-level-ish function bodies by brace depth
    (the report's paths are the GPU box's; the same file is looked up here)."""
    import pathlib
    local = list(pathlib.Path(__file__).resolve().parent.parent.rglob(pathlib.Path(path).name))
    try:
        src = open(local[0] if local else path).read().split("\n")
    except OSError:
        return []
    out, depth, cur, start = [], 0, None, 0
    sig = re.compile(r"^\s*(template\s*<.*>\s*)?(static\s+)?(__device__|__global__|PW_HD|PW_HD_COLD)[^;]*?(\w+)\s*\(")
    pending = None
    for i, line in enumerate(src, 1):
        m = sig.match(line)
        if m and depth <= 1:
            pending = (i, m.group(4))
        if "{" in line and pending and cur is None:
            cur, start = pending[1], pending[0]
            base = depth
        depth += line.count("{") - line.count("}")
        if cur is not None and depth <= base:
            out.append((start, i, cur))
            cur, pending = None, None
    return out


tot_i = sum(v[0] for v in per_line.values()) or 1
tot_s = sum(v[1] for v in per_line.values()) or 1
agg = defaultdict(lambda: [0, 0])
fcache = {}
for (f, ln), (i, s) in per_line.items():
    if f not in fcache:
        fcache[f] = functions(f) if "/cuda/" not in (f or "") else []
    name = next((n for a, b, n in fcache[f] if a <= ln <= b), None)
    key = f"{f.split('/')[-1]}:{name}" if name else f.split("/")[-1]
    agg[key][0] += i
    agg[key][1] += s
print(f"instructions {tot_i}  samples {tot_s}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{100 * i / tot_i:6.2f}%i {100 * s / tot_s:6.2f}%s  {k}")
