"""A/B timing of fixed operating points (kernel ms per 10K-query step), one
workload build shared by every library under test.

    python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 \
        --libs tools/lib_r01.so,default [--tuning JSON] [--rounds 2]

Each library is loaded as its own ctypes handle (its own copy of the
kernels); the shard is re-created from the same device tensors per library.
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import _abi, device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2s")
ap.add_argument("--l", type=int, default=160)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--tuning", default="", help="JSON object or list of objects")
ap.add_argument("--arms", default="naive,pathweaver")
ap.add_argument("--discard", type=float, default=0.5)
ap.add_argument("--ghost-iter", type=int, default=8)
ap.add_argument("--libs", default="default")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
tunings = json.loads(args.tuning) if args.tuning else [None]
if isinstance(tunings, dict):
    tunings = [tunings]
W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
gh = W["ghost"] or (None, None)
q = W["queries"]
default_path = _abi.LIB_PATH


def use_lib(path: str):
    _abi.LIB_PATH = default_path if path == "default" else Path(path)
    _abi._LIB = None
    return _abi.load()


for rnd in range(args.rounds):
    for lib_name in args.libs.split(","):
        lib = use_lib(lib_name)
        shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
        run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
        for tuning in tunings:
            out = {"lib": lib_name, "round": rnd, "tuning": tuning, "l": args.l}
            for arm, mode in (("naive", "baseline"), ("pathweaver", "pipelined")):
                if arm not in args.arms:
                    continue
                p = bench.arm_params(arm, args.l, cfg["k"], cfg.get("metric", "l2"), discard=args.discard,
                                     ghost_iter=args.ghost_iter)
                for _ in range(3):
                    dv.run_local([shard], p, q, mode, run, tuning=tuning)
                torch.cuda.synchronize()
                timer = []
                for _ in range(args.reps):
                    dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
                torch.cuda.synchronize()
                ms = sum(a.elapsed_time(b) for a, b in timer) / args.reps
                st = run.stats()[0]
                ids = run.final_ids.cpu().numpy()
                try:
                    lc = _abi.launch_config(shard.handle, p, tuning)
                except AttributeError:
                    lc = {"warps_per_sm": None, "smem_per_warp": None}
                out[arm] = dict(kernel_ms=round(ms, 3), qps=round(q.shape[0] / ms * 1e3),
                                warps=lc["warps_per_sm"], smem=lc["smem_per_warp"],
                                dc=float(st["distance_computations"].mean()), it=float(st["iterations"].mean()),
                                ids_sum=int(ids.astype("int64").sum()))
            print(json.dumps(out), flush=True)
        del shard, run
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
