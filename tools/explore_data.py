"""Exploration helper (not part of the product): data generators vs recall."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_17094_b200 import builder, device as dv, SearchParams

def arm(kind, l):
    if kind == "pw":
        return SearchParams(k=10, l=l, m=64, r=8, max_iter=64, seed=1, selection="direction",
                            discard_ratio=0.5, cooldown_ratio=0.3, ghost_enabled=True, ghost_max_iter=8)
    return SearchParams(k=10, l=l, m=64, r=8, max_iter=64, seed=1)

def trial(name, x, nq, j=32, probe=8):
    torch.cuda.synchronize(); t0 = time.time()
    base, q = x[:-nq].contiguous(), x[-nq:].contiguous()
    adj = builder.knn_graph(base, j, probe=probe)
    dr = builder.direction_table(base, adj)
    gh = builder.ghost(base, 0.01, 16, 0)
    torch.cuda.synchronize(); tb = time.time() - t0
    truth = builder.exact_knn_rescored(base, q, 10).cpu().numpy()
    sh = dv.TensorShard(base, adj, torch.arange(base.shape[0], device='cuda', dtype=torch.int32), dr, None, gh[0], gh[1])
    run = dv.DeviceRun(nq, 1, 10, 'cuda')
    res = {"name": name, "build_s": round(tb, 1)}
    for kind, mode in (("naive", "baseline"), ("pw", "pipelined")):
        rows = []
        for l in (32, 64, 96, 128, 192, 256, 384):
            p = arm(kind, l)
            dv.run_local([sh], p, q, mode, run)
            torch.cuda.synchronize()
            t = time.time(); reps = 3
            for _ in range(reps):
                dv.run_local([sh], p, q, mode, run)
            torch.cuda.synchronize(); dt = (time.time() - t) / reps
            rec = builder.recall_at_k(run.final_ids.cpu().numpy(), truth, 10)
            st = run.stats()[0]
            rows.append((l, round(rec, 4), int(nq / dt), int(st["distance_computations"].mean()), round(float(st["iterations"].mean()), 1)))
            if rec >= 0.97: break
        res[kind] = rows
    print(json.dumps(res), flush=True)

def graph_quality(x, j=32, sample=2000, probe=8):
    base = x
    torch.cuda.synchronize(); t0 = time.time()
    adj = builder.knn_graph(base, j, augment=False, probe=probe)
    torch.cuda.synchronize(); print('  knn build', probe, round(time.time()-t0, 2), flush=True)
    idx = torch.arange(0, base.shape[0], base.shape[0] // sample, device='cuda')[:sample]
    ex = builder.exact_knn(base, base[idx], j + 1)[:, 1:]
    a = adj[idx].long().cpu().numpy(); e = ex.cpu().numpy()
    return float(np.mean([len(set(p.tolist()) & set(q.tolist())) / j for p, q in zip(a, e)]))

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    nq = 10000
    x = builder.gen_latent(n + nq, 96, 16, 1, 1.0, 0.05, 7)
    for probe in (8, 16, 32, 64):
        print("lat16 probe", probe, "ivf graph recall", round(graph_quality(x[:-nq].contiguous(), probe=probe), 3), flush=True)
    trial("lat16-p32", x, nq, probe=32)
    x = builder.gen_latent(n + nq, 96, 12, 1, 1.0, 0.05, 7)
    trial("lat12-p32", x, nq, probe=32)
