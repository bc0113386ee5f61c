"""Profiling harness: build a bench workload and run one arm a few times so
ncu can capture a warm beam_search_kernel launch.

    ncu --set full --clock-control none --import-source on -k regex:beam_search \
        -s 2 -c 1 -o gpurun_out/prof python tools/profile_run.py --config c2s --arm pathweaver
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2s")
ap.add_argument("--arm", default="pathweaver")
ap.add_argument("--l", type=int, default=160)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--tuning", default="")
ap.add_argument("--discard", type=float, default=0.5)
ap.add_argument("--ghost-iter", type=int, default=8)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
run = dv.DeviceRun(W["queries"].shape[0], 1, cfg["k"], "cuda")
p = bench.arm_params(args.arm, args.l, cfg["k"], cfg.get("metric", "l2"), discard=args.discard,
                     ghost_iter=args.ghost_iter)
mode = "pipelined" if args.arm == "pathweaver" else "baseline"
import json
tuning = json.loads(args.tuning) if args.tuning else None
for _ in range(args.reps):
    dv.run_local([shard], p, W["queries"], mode, run, tuning=tuning)
torch.cuda.synchronize()
print("done", run.final_ids[0].tolist())
