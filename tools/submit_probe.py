"""Device-loop timing probe: K back-to-back RingSearch.submit batches (the
bench's `value` loop) with and without per-launch timers, final-id copies on
a side stream or in stream order.

    python tools/submit_probe.py --config c2s --l 96
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import device as dv, ring  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2s")
ap.add_argument("--l", type=int, default=96)
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
W = bench.build_workload(cfg, 0, 1, dev)
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q = W["queries"]
p = bench.arm_params("pathweaver", args.l, cfg["k"], cfg.get("metric", "l2"), discard=0.75, ghost_iter=1)
for side in (False, True, False, True):
    for with_timer in (False, True):
        eng = ring.RingSearch(shard, q.shape[0], cfg["k"], 0, 1, dev, tuning=json.loads(bench.DEFAULT_TUNING))
        eng.side_d2h = side
        for _ in range(3):
            eng.run(q, p, "pipelined")
        torch.cuda.synchronize()
        timers = [] if with_timer else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(args.steps):
            eng.submit(q, p, "pipelined", timer=timers)
        t1 = time.perf_counter()
        eng.sync()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        km = sum(a.elapsed_time(b) for a, b in timers) / args.steps if timers else None
        print(json.dumps(dict(side_d2h=side, timer=with_timer, ms_per_step=round(ms, 4), kernel_ms=km,
                              host_submit_ms=round((t1 - t0) * 1e3 / args.steps, 3))), flush=True)
