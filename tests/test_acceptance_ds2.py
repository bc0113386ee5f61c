"""End-to-end known-answer test on the reference's own acceptance dataset DS2
(tests/test_acceptance.py:39-41 of shardann: 100K x 32 points from
gen_synthetic(101000, 32, 6144, 0.055, seed=202), 4 shards, j=32,
rho=0.01, ghost degree 16, build seed 7; SearchParams(k=10, l=64, m=64, r=8,
max_iter=8, seed=11)).  The counters below are the reference's
(acceptance_report.txt, criteria 02/05/07); they depend on every generator
value, every index array, every distance bit and every RNG draw, so matching
them pins data -> exact GPU index build -> exact GPU ground truth -> K1 end
to end.  (SURVEY.md §8c names them as end-to-end KATs.)

CPU part: gen_synthetic reproduces the reference's generator bits (checked
against the conftest fixture the reference generated).
"""

from __future__ import annotations

import numpy as np
import pytest

import golden_util as gu
import paper_2507_17094_b200 as pw

# acceptance_report.txt (reference run): criterion 02 recall@10 at
# max_iter 8; criterion 07 total = discarded + retained; criterion 05 DGS
# distance computations and recall drops
RECALL = 0.9633
TOTAL_VISITS, RETAINED = 3_682_348, 256_000
DGS_COMPS, DGS_DROP, RND_DROP = 2_453_062, 0.0036, 0.0457


def test_gen_synthetic_matches_reference_fixture():
    z = gu.load("small")[0]
    full = pw.gen_synthetic(4100, 16, 32, 0.2, seed=99)  # conftest.py small_data
    assert np.array_equal(full.data[:4000], z["base"])
    assert np.array_equal(full.data[4000:], z["queries"])


@pytest.mark.gpu
def test_ds2_acceptance_counters():
    from paper_2507_17094_b200 import exact, metrics

    full = pw.gen_synthetic(101_000, 32, 6144, 0.055, seed=202)
    base = pw.Dataset(full.data[:100_000])
    queries = pw.Dataset(full.data[100_000:])
    index, _ = exact.build_index(base, 4, 32, seed=7, rho=0.01, ghost_degree=16)
    truth = metrics.exact_knn_batch(base, queries, 10)
    ctxs = pw.build_contexts(index, base)
    p = pw.SearchParams(k=10, l=64, m=64, r=8, max_iter=8, seed=11)

    res = pw.run_sharded_baseline(queries, index, base, p, contexts=ctxs)
    m = metrics.collect_metrics(res)
    recall = metrics.mean_recall(truth, res.neighbor_lists(), 10)
    assert recall == pytest.approx(RECALL, abs=1e-9)
    assert (m.total_visits, m.retained_visits) == (TOTAL_VISITS, RETAINED)
    assert m.discarded_visits == TOTAL_VISITS - RETAINED

    dgs = pw.run_sharded_baseline(queries, index, base,
                                  p.with_(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3),
                                  contexts=ctxs)
    assert metrics.collect_metrics(dgs).distance_computations == DGS_COMPS
    assert recall - metrics.mean_recall(truth, dgs.neighbor_lists(), 10) == pytest.approx(DGS_DROP, abs=1e-9)

    rnd = pw.run_sharded_baseline(queries, index, base,
                                  p.with_(selection="random", discard_ratio=0.5, cooldown_ratio=0.3),
                                  contexts=ctxs)
    assert recall - metrics.mean_recall(truth, rnd.neighbor_lists(), 10) == pytest.approx(RND_DROP, abs=1e-9)

    pipe = pw.run_pipelined(queries, index, base, p, contexts=ctxs)  # criterion 08
    assert np.all(pipe.comm_bytes_per_link == 3 * 250 * 4)
