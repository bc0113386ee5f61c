"""K4 tensor-core kNN screen: correctness against the FP32 screen and timing.

    python tools/knn_screen_probe.py [--n 200000] [--big 10000000]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2507_17094_b200 import builder, exact  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--big", type=int, default=0)
ap.add_argument("--big-rows", type=int, default=148 * 128 * 2)
ap.add_argument("--only-throughput", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
x = builder.gen_latent(args.n, args.d, 16, 1, 1.0, 0.05, 7, device=dev)

def checks():
    # 1. raw screen vs FP32 recomputation of the returned candidates
    q = x[:4096].contiguous()
    ids, vals, xn = exact.knn_screen_tc(x, q, 48, self_off=0)
    torch.cuda.synchronize()
    ok_ids = ids >= 0
    ref = xn[ids.clamp(min=0)] - 2.0 * (q[:, None, :] * x[ids.clamp(min=0)]).sum(-1)
    err = (vals - ref).abs()[ok_ids]
    bound = exact.TC_ERR * q.norm(dim=1)[:, None] * x[ids.clamp(min=0)].norm(dim=2)
    print(json.dumps({"check": "screen values", "max_abs_err": float(err.max()),
                      "max_err_over_bound": float((err / bound[ok_ids]).max()),
                      "self_in_list": int((ids == torch.arange(4096, device=dev)[:, None]).sum()),
                      "full_rows": int(ok_ids.all(1).sum())}), flush=True)
    # 2. exact top-k through the tc screen (certified) == through the FP32 screen
    st = {}
    t0 = time.perf_counter()
    a_ids, a_sq = exact.exact_topk(x, q, 32, exclude_self=False, screen="tc", stats=st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b_ids, b_sq = exact.exact_topk(x, q, 32, exclude_self=False, screen="fp32")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"check": "exact_topk tc == fp32", "ids_equal": bool(torch.equal(a_ids, b_ids)),
                      "sq_equal": bool(torch.equal(a_sq, b_sq)), "stats": st,
                      "tc_s": round(t1 - t0, 3), "fp32_s": round(t2 - t1, 3)}), flush=True)
    g_tc = exact.build_knn_graph(x[:60000].contiguous(), 32)  # auto -> fp32 (small)
    st2 = {}
    a2, _ = exact.exact_topk(x[:60000].contiguous(), x[:60000].contiguous(), 32, exclude_self=True, screen="tc",
                             stats=st2)
    b2, _ = exact.exact_topk(x[:60000].contiguous(), x[:60000].contiguous(), 32, exclude_self=True, screen="fp32")
    print(json.dumps({"check": "self-excluded graph rows tc == fp32", "ids_equal": bool(torch.equal(a2, b2)),
                      "stats": st2}), flush=True)


if not args.only_throughput:
    checks()
# 3. throughput of the screen alone: query rows x all base rows
for n in ([args.n] + ([args.big] if args.big else [])):
    xb = x if n == args.n else builder.gen_latent(n, args.d, 16, 1, 1.0, 0.05, 8, device=dev)
    qq = xb[: min(args.big_rows, n)].contiguous()
    exact.knn_screen_tc(xb, qq[:128], 48, self_off=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    exact.knn_screen_tc(xb, qq, 48, self_off=0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    pairs = qq.shape[0] * n
    tflops = 2.0 * pairs * args.d / (ms / 1e3) / 1e12
    print(json.dumps({"check": "screen throughput", "n": n, "query_rows": qq.shape[0], "ms": round(ms, 2),
                      "tflops_tf32": round(tflops, 1),
                      "projected_full_graph_s": round(ms / 1e3 * n / qq.shape[0], 1)}), flush=True)
