"""Hot SASS regions of an ncu report: per-instruction executed counts and
stall samples, printed as address ranges ordered by instructions.

    python tools/sass_hot.py gpurun_out/prof.ncu-rep [min_share]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ia, isrc, isamp, iinst = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    ins.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iinst] or 0)))
tot_i = sum(x[3] for x in ins)
tot_s = sum(x[2] for x in ins)
base = ins[0][0]
print(f"instructions {tot_i}  samples {tot_s}  sass lines {len(ins)}")
# print every instruction with >= thr share of instructions or samples, plus 2 lines of context
keep = set()
for k, x in enumerate(ins):
    if x[3] >= thr * tot_i or x[2] >= thr * tot_s:
        keep.update(range(max(0, k - 1), min(len(ins), k + 2)))
last = -2
for k in sorted(keep):
    if k != last + 1:
        print("   ...")
    a, src, s, i = ins[k]
    print(f"{a - base:6x} {100 * i / tot_i:5.2f}%i {100 * s / tot_s:5.2f}%s  {src}")
    last = k
