"""A/B of the end-to-end C-ABI call (pw_run with pinned host buffers) across
library builds, with a GPU timeline of one call per library: where the
e2e time goes between the call's entry, the first copy, K1, K2, the result
copies and the call's return.

    python tools/e2e_ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 \
        --libs tools/lib_prev.so,default [--steps 20] [--rounds 2]
"""
import argparse
import gc
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile, record_function  # noqa: E402

import bench  # noqa: E402
from paper_2507_17094_b200 import _abi, builder, device as dv, ring  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--l", type=int, default=112)
ap.add_argument("--discard", type=float, default=0.75)
ap.add_argument("--ghost-iter", type=int, default=1)
ap.add_argument("--libs", default="default")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=2)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
W = bench.build_workload(cfg, 0, 1, dev)
gh = W["ghost"] or (None, None)
nq = W["queries"].shape[0]
qh = torch.empty(tuple(W["queries"].shape), dtype=W["queries"].dtype, pin_memory=True)
qh.copy_(W["queries"].cpu())
qh = qh.numpy()
default_path = _abi.LIB_PATH
truth = bench.ground_truth(W, cfg["k"], cfg.get("metric", "l2"))
torch.cuda.empty_cache()  # the truth's cached blocks would starve pw_shard_create's cudaMalloc
p = bench.arm_params("pathweaver", args.l, cfg["k"], cfg.get("metric", "l2"), discard=args.discard,
                     ghost_iter=args.ghost_iter)


def use_lib(path):
    # "<lib>+nostream": the same library with pw_run's streamed download off
    path, _, opt = path.partition("+")
    if opt == "nostream":
        os.environ["PW_NO_STREAM_OUT"] = "1"
    else:
        os.environ.pop("PW_NO_STREAM_OUT", None)
    _abi.LIB_PATH = default_path if path == "default" else Path(path)
    _abi._LIB = None
    return _abi.load()


def timeline(eng):
    """GPU activity of the middle of three profiled calls, relative to the
    call's host entry (us)."""
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(3):
            with record_function(f"call{i}"):
                eng.run_host(qh, p)
        torch.cuda.synchronize()
    path = Path(tempfile.mkdtemp()) / "t.json"
    prof.export_chrome_trace(str(path))
    ev = json.loads(path.read_text())["traceEvents"]
    call = [e for e in ev if e.get("name") == "call1" and e.get("cat") == "user_annotation"][0]
    t0, t1 = call["ts"], call["ts"] + call["dur"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and t0 <= e["ts"] <= t1]
    out = []
    for e in sorted(gpu, key=lambda e: e["ts"]):
        name = e["name"]
        if e["cat"] == "kernel":
            name = "K1" if "beam_search" in name else ("K2" if "reduce_topk" in name else name[:40])
        out.append((round(e["ts"] - t0, 1), round(e["dur"], 1), e["cat"].replace("gpu_", ""), name[:40]))
    return round(call["dur"], 1), out


for rnd in range(args.rounds):
    for lib_name in args.libs.split(","):
        use_lib(lib_name)
        shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
        eng = ring.RingSearch(shard, nq, cfg["k"], 0, 1, dev, tuning={"flags": 2})
        for _ in range(3):
            eng.run_host(qh, p)
        t = time.perf_counter()
        for _ in range(args.steps):
            res = eng.run_host(qh, p)
        dt = (time.perf_counter() - t) / args.steps
        rec = {"lib": lib_name, "round": rnd, "ms_per_call": round(dt * 1e3, 4), "e2e_qps": round(nq / dt, 1),
               "recall": round(builder.recall_at_k(res["final_ids"], truth, 10), 4)}
        if rnd == args.rounds - 1:
            dur, tl = timeline(eng)
            rec["call_us"] = dur
            rec["timeline"] = tl
        print(json.dumps(rec), flush=True)
        del eng, shard, res
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
