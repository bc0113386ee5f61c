"""K1 time vs batch size at one operating point: how much of a step is the
last, partly-occupied wave of the persistent kernel (tail).

    python tools/tail_probe.py --config c2 --l 256
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import _abi, device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--l", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--discard", type=float, default=0.75)
ap.add_argument("--ghost-iter", type=int, default=1)
ap.add_argument("--tuning", default='{"flags": 2}')
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tuning = json.loads(args.tuning)
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q_all = W["queries"]
for arm, mode in (("pathweaver", "pipelined"), ("naive", "baseline")):
    p = bench.arm_params(arm, args.l, cfg["k"], discard=args.discard, ghost_iter=args.ghost_iter)
    lc = _abi.launch_config(shard.handle, p, tuning)
    warps = lc["warps_per_sm"] * lc["blocks"]
    for mult in (1, 2, 3, 4, None, 8):
        q = q_all if mult is None else torch.cat([q_all] * 3)[: warps * mult]
        run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
        for _ in range(2):
            dv.run_local([shard], p, q, mode, run, tuning=tuning)
        torch.cuda.synchronize()
        timer = []
        for _ in range(args.reps):
            dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in timer) / args.reps
        print(json.dumps({"arm": arm, "queries": q.shape[0], "waves": round(q.shape[0] / warps, 2),
                          "kernel_ms": round(ms, 3), "us_per_query": round(ms * 1e3 / q.shape[0], 4)}),
              flush=True)
