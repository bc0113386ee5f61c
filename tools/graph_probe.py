"""Graph quality vs the IVF builder's probe count, and what it does to both
arms' operating points (C2).  The reference builds an exact kNN graph
(graphs.py:104-134); a closer approximation is a closer workload.

    python tools/graph_probe.py --probes 48,96,192
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
from paper_2507_17094_b200 import builder, device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--probes", default="48,96,192")
ap.add_argument("--refines", default="0")
args = ap.parse_args()
tuning = {"flags": 2}
for probe, refine in ((int(p), int(r)) for p in args.probes.split(",") for r in args.refines.split(",")):
    cfg = dict(bench.CONFIGS[args.config], probe=probe, refine=refine)
    t0 = time.time()
    W = bench.build_workload(cfg, 0, 1, torch.device("cuda", 0))
    build_s = time.time() - t0
    truth = bench.ground_truth(W, cfg["k"])
    # graph accuracy: the first j entries of 2000 rows vs the exact j-NN
    x = W["vec"]
    rows = torch.arange(0, x.shape[0], x.shape[0] // 2000, device=x.device)[:2000]
    ex = builder.exact_knn(x, x[rows], cfg["j"] + 1)[:, 1:]
    got = W["adj"][rows, : cfg["j"]].long()
    acc = float((got.unsqueeze(2) == ex.unsqueeze(1)).any(2).float().mean())
    gh = W["ghost"] or (None, None)
    shard = dv.TensorShard(W["vec"], W["adj"], W["rows"].to(torch.int32), W["direction"], None, gh[0], gh[1])
    q = W["queries"]
    run = dv.DeviceRun(q.shape[0], 1, cfg["k"], "cuda")
    out = {"probe": probe, "refine": refine, "build_s": round(build_s, 1), "graph_recall_at_j": round(acc, 4)}
    for arm, mode, kw in (("naive", "baseline", {}), ("pathweaver", "pipelined", dict(discard=0.8, ghost_iter=1))):
        for l in bench.L_GRID:
            p = bench.arm_params(arm, l, cfg["k"], **kw)
            dv.run_local([shard], p, q, mode, run, tuning=tuning)
            torch.cuda.synchronize()
            rec = builder.recall_at_k(run.final_ids.cpu().numpy(), truth, 10)
            if rec >= 0.95:
                break
        timer = []
        for _ in range(2):
            dv.run_local([shard], p, q, mode, run, tuning=tuning)
        for _ in range(5):
            dv.run_local([shard], p, q, mode, run, tuning=tuning, timer=timer)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in timer) / 5
        out[arm] = {"l": l, "recall": round(rec, 4), "ms": round(ms, 3)}
    print(json.dumps(out), flush=True)
    del W, shard, run
    torch.cuda.empty_cache()
