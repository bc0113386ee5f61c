"""Operating points for arbitrary SearchParams variants: for each variant the
smallest l (grid) reaching recall@10 >= 0.95 and its K1 time.

    python tools/explore_variants.py --config c2 --arm pathweaver \
        --variants '[{"discard_ratio": 0.8}, {"discard_ratio": 0.8, "m": 32}]'
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
ap.add_argument("--arm", default="pathweaver")
ap.add_argument("--variants", required=True)
ap.add_argument("--grid", default="128,160,192,224,256,288,320,384")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tuning = {"flags": 2}
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
truth = bench.ground_truth(W, cfg["k"])
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q = W["queries"]
run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
mode = "pipelined" if args.arm == "pathweaver" else "baseline"
for var in json.loads(args.variants):
    best = None
    for l in (int(x) for x in args.grid.split(",")):
        p = dataclasses.replace(bench.arm_params(args.arm, l, cfg["k"]), **var)
        dv.run_local([shard], p, q, mode, run, tuning=tuning)
        torch.cuda.synchronize()
        rec = builder.recall_at_k(run.final_ids.cpu().numpy(), truth, 10)
        if rec >= 0.95:
            best = (p, rec)
            break
    if best is None:
        print(json.dumps({"variant": var, "reached": False}), flush=True)
        continue
    p, rec = best
    timer = []
    for _ in range(2):
        dv.run_local([shard], p, q, mode, run, tuning=tuning)
    for _ in range(5):
        dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in timer) / 5
    print(json.dumps({"variant": var, "l": p.l, "recall": round(rec, 4), "kernel_ms": round(ms, 3),
                      "qps": round(q.shape[0] / ms * 1e3)}), flush=True)
