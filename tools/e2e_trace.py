"""CUPTI trace (torch.profiler) of the end-to-end C-ABI call (pw_run with
pinned host buffers) to see where the e2e overhead goes.

    python tools/e2e_trace.py --config c4 --l 80
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import device as dv, ring  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--l", type=int, default=80)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
W = bench.build_workload(cfg, 0, 1, dev)
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
eng = ring.RingSearch(shard, W["queries"].shape[0], cfg["k"], 0, 1, dev, tuning={"flags": 2})
p = bench.arm_params("pathweaver", args.l, cfg["k"], cfg.get("metric", "l2"), discard=0.8, ghost_iter=1)
qh = torch.empty(tuple(W["queries"].shape), dtype=torch.float32, pin_memory=True)
qh.copy_(W["queries"].cpu())
qh = qh.numpy()
for _ in range(3):
    eng.run_host(qh, p)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        eng.run_host(qh, p)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=15))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
