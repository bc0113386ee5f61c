"""Minimal repro of the TMA gather4 scoring path on the parity fixture."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import oracle
import paper_2507_17094_b200 as pw
from golden_util import oracle_dict, result_dict, assert_run_equal, assert_run_equal_lossy
from index_util import clustered, make_contexts
from paper_2507_17094_b200.search import SearchParams

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x = clustered(24000 + 600, 96, 512, 0.08, seed=96)
q, ctxs = np.ascontiguousarray(x[24000:24000 + nq]), make_contexts(x[:24000], 2, 32, seed=96)
p = SearchParams(k=10, l=64, m=64, r=8, max_iter=64, seed=1)
got = result_dict(pw.run_sharded_baseline(pw.Dataset(q), None, None, p, contexts=ctxs, tuning={"flags": flags}))
want = oracle_dict(oracle.run(q, ctxs, p, "baseline"))
(assert_run_equal_lossy if flags & 2 else assert_run_equal)(got, want, "repro")
print("ok", flags, nq)
