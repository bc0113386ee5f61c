"""Exact kNN graph (graphs.py:104-134 semantics) at bench scale with the K4
tensor-core screen: time per phase, certification, and the share of each
row's exact 32-NN that the approximate IVF builder keeps.

    python tools/exact_build_probe.py --config c2
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
from paper_2507_17094_b200 import builder, exact  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--compare-ivf", action="store_true")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
x = builder.gen_latent(cfg["n"] + cfg["nq"], cfg["d"], cfg["m"], cfg["n_clusters"], cfg["spread"], cfg["noise"],
                       bench.SEED, device=dev)
if cfg.get("dtype") == "u8":
    x = torch.clamp(torch.round(128.0 + 40.0 * x), 0, 255)
if cfg.get("metric") == "ip":
    x = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
base = x[: cfg["n"]].contiguous()
del x
torch.cuda.synchronize()
st = {}
t0 = time.perf_counter()
adj = exact.build_knn_graph(base, cfg["j"], stats=st)
torch.cuda.synchronize()
st["total_s"] = round(time.perf_counter() - t0, 2)
out = {"config": args.config, "n": cfg["n"], "d": cfg["d"], "exact": st,
       "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}
if args.compare_ivf:
    t1 = time.perf_counter()
    ivf = builder.knn_graph(base, cfg["j"], probe=cfg["probe"], seed=bench.SEED, refine=cfg.get("refine", 0))
    torch.cuda.synchronize()
    out["ivf_s"] = round(time.perf_counter() - t1, 1)
    # share of each row's exact (pre-augmentation proxy: the augmented row) ids the IVF graph holds
    rows = torch.randint(0, cfg["n"], (20000,), device=dev)
    a, b = adj[rows].long(), ivf[rows].long()
    hit = (a[:, :, None] == b[:, None, :]).any(2).float().mean()
    out["ivf_share_of_exact_rows"] = round(float(hit), 4)
print(json.dumps(out), flush=True)
