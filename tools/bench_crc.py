"""K3 (device CRC-32C of container sections) vs the host CRC on this box.

    python tools/bench_crc.py [--gb 4]
Prints GB/s of one K3 launch over a buffer larger than L2 (CUDA events on the
launch stream) against MEASURED_PEAKS.json's HBM figure, and the host path.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2507_17094_b200 as pw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
ap.add_argument("--sections", type=int, default=7)
args = ap.parse_args()
n = int(args.gb * 1e9)
buf = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
cuts = torch.linspace(0, n, args.sections + 1).long().tolist()
secs = [buf[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
st = torch.cuda.current_stream()
pw.crc32c_device(secs)
times = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    got = pw.crc32c_device(secs)  # synchronous: one K3 launch + 28-byte readback
    e1.record(st)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = sorted(times)[len(times) // 2]
# kernel-only duration from CUPTI activity records (torch.profiler; no replay)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        pw.crc32c_device(secs)
    torch.cuda.synchronize()
kus = [e.device_time for e in prof.events() if "crc32c_sections_kernel" in e.name]
kms = (sorted(kus)[len(kus) // 2] / 1e3) if kus else None
host = buf[: min(n, 1 << 30)].cpu().numpy()
t0 = time.perf_counter()
hc = pw.crc32c(host)
hs = time.perf_counter() - t0
assert pw.crc32c_device([buf[: host.size]]) == [hc]
try:
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0)
except OSError:
    peak = 6650.0
dev_gbs = n / (ms / 1e3) / 1e9
print(json.dumps({"kernel": "crc32c_sections_kernel", "bytes": n, "sections": args.sections,
                  "kernel_ms": None if kms is None else round(kms, 3),
                  "kernel_gbs": None if kms is None else round(n / (kms / 1e3) / 1e9, 1),
                  "kernel_frac": None if kms is None else round(n / (kms / 1e3) / 1e9 / peak, 3),
                  "ms_per_call_incl_setup_readback": round(ms, 3), "call_gbs": round(dev_gbs, 1),
                  "peak_gbs": peak, "call_frac": round(dev_gbs / peak, 3),
                  "host_gbs": round(host.size / hs / 1e9, 2), "host_threads": os.cpu_count()}))
