"""Per-phase cycle breakdown of K1 (needs libpwb200_timers.so: PW_LIB=...).

    python -m paper_2507_17094_b200.build_ext --timers
    PW_LIB=paper_2507_17094_b200/libpwb200_timers.so python tools/phase_timers.py --config c2 --l 256
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import _abi, device as dv  # noqa: E402

PHASES = ("init", "score", "merge", "select", "expand", "dedup", "visited", "other")
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--l", type=int, default=256)
ap.add_argument("--tuning", default="")
ap.add_argument("--discard", type=float, default=0.5)
ap.add_argument("--ghost-iter", type=int, default=8)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tuning = json.loads(args.tuning) if args.tuning else None
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
gh = W["ghost"] or (None, None)
shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
q = W["queries"]
run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
lib = _abi.load()
out = (C.c_int64 * 8)()
for arm, mode in (("pathweaver", "pipelined"), ("naive", "baseline")):
    p = bench.arm_params(arm, args.l, cfg["k"], discard=args.discard, ghost_iter=args.ghost_iter)
    dv.run_local([shard], p, q, mode, run, tuning=tuning)
    torch.cuda.synchronize()
    _abi.check(lib.pw_phase_cycles(shard.handle, out, 1))
    dv.run_local([shard], p, q, mode, run, tuning=tuning)
    torch.cuda.synchronize()
    _abi.check(lib.pw_phase_cycles(shard.handle, out, 1))
    cyc = np.array(list(out), dtype=np.float64)
    st = run.stats()[0]
    iters = float(st["iterations"].sum() + st["ghost_iterations"].sum())
    lc = _abi.launch_config(shard.handle, p, tuning)
    warps = lc["warps_per_sm"] * lc["blocks"]
    print(json.dumps({"arm": arm, "l": args.l, "iterations": iters, "warps": warps,
                      "cycles_per_iteration": round(cyc.sum() / iters, 1),
                      "share": {ph: round(c / cyc.sum(), 4) for ph, c in zip(PHASES, cyc)},
                      "cycles_per_iter_by_phase": {ph: round(c / iters, 1) for ph, c in zip(PHASES, cyc)}}),
          flush=True)
