"""pw_run's overlapped query upload with pageable and page-locked queries."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch
import paper_2507_17094_b200 as pw
from index_util import clustered, make_contexts
from paper_2507_17094_b200.search import SearchParams

import time
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
tun = {"flags": int(sys.argv[2])} if len(sys.argv) > 2 else None
x = clustered(20000 + nq, 96, 256, 0.08, seed=3)
ctxs = make_contexts(x[:20000], 1, 32, seed=3)
p = SearchParams(k=10, l=64, m=64, r=8, max_iter=32, seed=1, selection="direction", discard_ratio=0.75,
                 ghost_enabled=True, ghost_max_iter=1)
q = np.ascontiguousarray(x[20000:])
t0 = time.time()
r1 = pw.run_pipelined(pw.Dataset(q), None, None, p, contexts=ctxs, tuning=tun)
print("t", time.time() - t0)
print("pageable ok", r1.final_ids[:2, :3].tolist(), flush=True)
qp = torch.empty(q.shape, dtype=torch.float32, pin_memory=True).numpy()
qp[:] = q
t0 = time.time()
r2 = pw.run_pipelined(pw.Dataset(qp), None, None, p, contexts=ctxs, tuning=tun)
print("t", time.time() - t0)
print("pinned ok", np.array_equal(r1.final_ids, r2.final_ids), flush=True)
