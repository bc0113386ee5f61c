"""Basic-block view of an ncu source capture: runs of SASS with the same
execution count, their instruction share, stall share and the CUDA source
lines they come from.

    python tools/ncu_blocks.py gpurun_out/prof.ncu-rep [min_share] [n_queries]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
nq = float(sys.argv[3]) if len(sys.argv) > 3 else 10000.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
# mixed view: CUDA line rows ("Line No" header) followed by their SASS rows?  ncu prints
# per file: CUDA lines with aggregated metrics; the SASS listing comes with --print-source sass.
txt2 = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
r2 = list(csv.reader(io.StringIO(txt2)))
hdr = r2[1]
ia, isrc, isamp, iinst = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                  "Instructions Executed"))
ins = [(int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iinst] or 0)) for r in r2[2:] if len(r) >= len(hdr)]
# address -> cuda line via the correlation in --print-source sass,cuda is not in CSV; use the
# source page with "cuda,sass": rows after a CUDA line row list that line's SASS addresses.
line_of = {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].strip().isdigit():
        cur = f"{fname}:{r[0].strip()}"
    elif r[0].startswith("0x") and cur:
        line_of[int(r[0], 16)] = cur
tot_i = sum(x[3] for x in ins) or 1
tot_s = sum(x[2] for x in ins) or 1
base = ins[0][0]
blocks, b = [], None
for a, src, s, i in ins:
    if b and b["i"] == i:
        b["n"] += 1
        b["s"] += s
        b["lines"][line_of.get(a, "?")] += 1
    else:
        b = {"a": a, "i": i, "n": 1, "s": s, "lines": Counter([line_of.get(a, "?")])}
        blocks.append(b)
print(f"instructions {tot_i} ({tot_i / nq:.0f}/query)  samples {tot_s}")
for b in sorted(blocks, key=lambda b: -b["i"] * b["n"]):
    share = b["i"] * b["n"] / tot_i
    if share < thr:
        break
    top = ", ".join(f"{k}x{v}" for k, v in b["lines"].most_common(4))
    print(f"{b['a'] - base:6x} n={b['n']:4d} x{b['i'] / nq:7.1f}/q {100 * share:5.2f}%i {100 * b['s'] / tot_s:5.2f}%s  {top}")
