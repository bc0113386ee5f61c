"""Operating-point search beyond l: for each arm and each (r, discard) pair,
the smallest l reaching recall@10 >= 0.95 and its K1 time.

    python tools/explore_params.py --config c2
"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import builder, device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--rs", default="4,8,16")
ap.add_argument("--discards", default="0.5,0.3,0.7")
ap.add_argument("--cooldowns", default="0.3")
ap.add_argument("--grid", default="")
ap.add_argument("--arms", default="pathweaver,naive")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tuning = {"flags": 2}
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
truth = bench.ground_truth(W, cfg["k"])
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q = W["queries"]
run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
grid = [int(x) for x in args.grid.split(",")] if args.grid else [l for l in bench.L_GRID if l >= cfg["k"]]


def timed(p, mode):
    for _ in range(2):
        dv.run_local([shard], p, q, mode, run, tuning=tuning)
    torch.cuda.synchronize()
    timer = []
    for _ in range(5):
        dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in timer) / 5


for arm, mode in (("pathweaver", "pipelined"), ("naive", "baseline")):
    if arm not in args.arms:
        continue
    discards = [float(x) for x in args.discards.split(",")] if arm == "pathweaver" else [None]
    cools = [float(x) for x in args.cooldowns.split(",")] if arm == "pathweaver" else [None]
    for r, dr, cr in ((r, dr, cr) for r in (int(x) for x in args.rs.split(",")) for dr in discards for cr in cools):
        if True:
            best = None
            for l in grid:
                if l < r:
                    continue
                p = bench.arm_params(arm, l, cfg["k"])
                p = dataclasses.replace(p, r=r) if dr is None else dataclasses.replace(p, r=r, discard_ratio=dr, cooldown_ratio=cr)
                try:
                    dv.run_local([shard], p, q, mode, run, tuning=tuning)
                except Exception as e:  # noqa: BLE001 -- configuration too large for shared memory
                    print(json.dumps({"arm": arm, "r": r, "discard": dr, "cooldown": cr, "l": l, "error": str(e)[:80]}), flush=True)
                    break
                torch.cuda.synchronize()
                rec = builder.recall_at_k(run.final_ids.cpu().numpy(), truth, 10)
                if rec >= 0.95:
                    best = (l, rec)
                    break
            if best is None:
                print(json.dumps({"arm": arm, "r": r, "discard": dr, "cooldown": cr, "reached": False}), flush=True)
                continue
            p = bench.arm_params(arm, best[0], cfg["k"])
            p = dataclasses.replace(p, r=r) if dr is None else dataclasses.replace(p, r=r, discard_ratio=dr, cooldown_ratio=cr)
            ms = timed(p, mode)
            print(json.dumps({"arm": arm, "r": r, "discard": dr, "cooldown": cr, "l": best[0], "recall": round(best[1], 4),
                              "kernel_ms": round(ms, 3), "qps": round(q.shape[0] / ms * 1e3)}), flush=True)
