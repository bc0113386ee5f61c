"""A/B timing of fixed operating points (kernel ms per 10K-query step).

    PW_LIB=path/to/lib.so python tools/ab.py --config c2s --l 160 [--tuning JSON]
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import builder, device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2s")
ap.add_argument("--l", type=int, default=160)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tuning", default="", help="JSON object or list of objects")
ap.add_argument("--arms", default="naive,pathweaver")
ap.add_argument("--discard", type=float, default=0.5)
ap.add_argument("--ghost-iter", type=int, default=8)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tunings = json.loads(args.tuning) if args.tuning else [None]
if isinstance(tunings, dict):
    tunings = [tunings]
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q = W["queries"]
run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
for tuning in tunings:
    out = {"lib": os.environ.get("PW_LIB", "default"), "tuning": tuning, "l": args.l}
    for arm, mode in (("naive", "baseline"), ("pathweaver", "pipelined")):
        if arm not in args.arms:
            continue
        p = bench.arm_params(arm, args.l, cfg["k"], discard=args.discard, ghost_iter=args.ghost_iter)
        for _ in range(3):
            dv.run_local([shard], p, q, mode, run, tuning=tuning)
        torch.cuda.synchronize()
        timer = []
        for _ in range(args.reps):
            dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in timer) / args.reps
        st = run.stats()[0]
        from paper_2507_17094_b200 import _abi
        try:
            lc = _abi.launch_config(shard.handle, p, tuning)
        except AttributeError:
            lc = {"warps_per_sm": None, "smem_per_warp": None}
        out[arm] = dict(kernel_ms=round(ms, 3), qps=round(q.shape[0] / ms * 1e3),
                        warps=lc["warps_per_sm"], smem=lc["smem_per_warp"],
                        dc=float(st["distance_computations"].mean()), it=float(st["iterations"].mean()))
    print(json.dumps(out), flush=True)
