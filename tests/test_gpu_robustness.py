"""Robustness of the C ABI: index validation, K2 tie order, device-side
reduce errors, and concurrent searches on one shard."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import paper_2507_17094_b200 as pw
from golden_util import load
from paper_2507_17094_b200 import device as dv
from paper_2507_17094_b200.rng import TAG_SEARCH, stream
from paper_2507_17094_b200.search import SearchParams, ShardContext

pytestmark = pytest.mark.gpu


def _ctx(vectors, adj, **kw):
    return ShardContext(vectors=vectors, adj=adj, global_ids=np.arange(vectors.shape[0], dtype=np.int32), **kw)


def test_reduce_topk_equal_keys_keep_every_copy():
    """np.lexsort is stable: equal (dist, id) candidates all survive
    (pipeline.py:195); ranks must not collide."""
    ids, dists = pw.reduce_topk(np.array([1, 1, 2]), np.array([0.5, 0.5, 0.7], np.float32), 3)
    assert ids.tolist() == [1, 1, 2]
    assert dists.tolist() == [0.5, 0.5, np.float32(0.7)]
    ids, _ = pw.reduce_topk(np.array([4, 4, 4, -1]), np.array([1, 1, 1, np.inf], np.float32), 2)
    assert ids.tolist() == [4, 4]


@pytest.mark.parametrize("bad", [-1, 10, 1 << 20])
def test_adjacency_ids_out_of_range_rejected(bad):
    x = np.arange(10, dtype=np.float32)[:, None]
    adj = np.zeros((10, 2), np.int32)
    adj[7, 1] = bad
    ctx = _ctx(x, adj)
    params = SearchParams(k=1, l=4, m=4, r=1, max_iter=4, seed=0)
    with pytest.raises(ValueError, match="adjacency id .* outside shard of 10 nodes"):
        pw.search(np.zeros(1, np.float32), ctx, params, rng=stream(0, TAG_SEARCH, 0, 0))


def test_ghost_ids_out_of_range_rejected():
    from paper_2507_17094_b200.search import GhostContext
    x = np.arange(40, dtype=np.float32)[:, None]
    adj = np.zeros((40, 2), np.int32)
    gids = np.array([0, 5, 50], np.int32)  # 50 >= n
    gh = GhostContext(vectors=x[[0, 5, 0]], adj=np.zeros((3, 1), np.int32), parent_ids=gids)
    with pytest.raises(ValueError, match="ghost parent id 50"):
        pw.search(np.zeros(1, np.float32), _ctx(x, adj, ghost=gh), SearchParams(k=1, l=4, m=4, r=1,
                  max_iter=4, seed=0), rng=stream(0, TAG_SEARCH, 0, 0))
    gh = GhostContext(vectors=x[[0, 5, 9]], adj=np.array([[1], [2], [3]], np.int32),
                      parent_ids=np.array([0, 5, 9], np.int32))  # ghost-local id 3 >= g
    with pytest.raises(ValueError, match="ghost adjacency id 3"):
        pw.search(np.zeros(1, np.float32), _ctx(x, adj, ghost=gh), SearchParams(k=1, l=4, m=4, r=1,
                  max_iter=4, seed=0), rng=stream(0, TAG_SEARCH, 0, 0))


def test_inter_map_out_of_range_rejected():
    """inter_map values seed the next shard (pipeline.py:339): validated
    against that shard's size before any pipelined launch."""
    z, base, queries, index, ctxs = load("small")
    shards = []
    for i, p in enumerate(index.shards):
        inter = p.inter_map.copy()
        if i == 1:
            inter[3] = 10 ** 6
        shards.append(pw.ShardPack(p.global_ids, p.adj, inter, p.ghost_ids, p.ghost_adj, p.direction))
    bad = pw.Index(d=index.d, n_total=index.n_total, shards=shards)
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17)
    with pytest.raises(ValueError, match="inter-shard map id 1000000"):
        pw.run_pipelined(pw.Dataset(queries), bad, base, params)
    # the baseline never reads inter_map
    res = pw.run_sharded_baseline(pw.Dataset(queries), bad, base, params)
    assert res.final_ids.shape == (queries.shape[0], 10)


def test_device_reduce_flag_raises():
    """The device-resident paths hand K2 a flag instead of synchronising;
    it is read where the results come back and raises like pipeline.py:194."""
    run = dv.DeviceRun(3, 2, 4, "cuda")
    run.reset()
    run.shard_ids[0].fill_(5)
    run.shard_dists[0].fill_(1.0)
    dv.reduce(run)
    with pytest.raises(ValueError, match="cannot reduce empty candidate lists"):
        run.check()
    run.check()  # the flag was cleared
    run.shard_ids.fill_(5)
    run.shard_dists.fill_(1.0)
    dv.reduce(run)
    run.check()
    assert run.final_ids.cpu().numpy().tolist() == [[5] * 4] * 3


def test_concurrent_searches_on_one_shard_match_serial():
    """search() is reentrant in the reference (pipeline.py drives it from a
    ThreadPoolExecutor): concurrent calls on one shard must not share a
    launch's task counter / visited tables."""
    z, base, queries, index, ctxs = load("small")
    ctx = pw.build_contexts(index, base)[0]
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17, selection="direction",
                          discard_ratio=0.5)

    def one(qi):
        res = pw.search(queries[qi], ctx, params, rng=stream(17, TAG_SEARCH, qi, 0), query_id=qi)
        return res.ids.tolist(), res.dists.tolist(), res.counters.distance_computations

    serial = [one(qi) for qi in range(48)]
    with ThreadPoolExecutor(8) as ex:
        for _ in range(3):
            assert list(ex.map(one, range(48))) == serial
    torch.cuda.synchronize()


def test_init_outputs_one_launch():
    """pw_init_outputs (DeviceRun.reset): padding ids -1, distances +inf,
    StageStats zero, whatever the buffers held before."""
    run = dv.DeviceRun(257, 3, 7, "cuda")
    for t in (run.shard_ids, run.s32, run.s64):
        t.fill_(12345)
    run.shard_dists.fill_(0.5)
    run.reset()
    torch.cuda.synchronize()
    assert bool((run.shard_ids == -1).all()) and bool(torch.isinf(run.shard_dists).all())
    assert int(run.s32.abs().sum()) == 0 and int(run.s64.abs().sum()) == 0


def test_submit_batches_equal_run():
    """RingSearch.submit (the bench's device loop: final-id copies on a side
    stream, the next batch's reduce ordered after the previous copy) returns
    the same ids as the synchronous run, batch after batch, alternating
    parameter sets."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).parent))
    from df_util import tensor_shard
    from paper_2507_17094_b200 import ring

    z, base, queries, index, ctxs = load("small")
    shard = tensor_shard(ctxs[0])
    q = torch.from_numpy(np.ascontiguousarray(queries)).cuda()
    eng = ring.RingSearch(shard, q.shape[0], 10, 0, 1, "cuda", tuning={"flags": 2})
    pa = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17)
    pb = SearchParams(k=10, l=48, m=32, r=4, max_iter=24, seed=5, selection="direction", discard_ratio=0.5)
    want = {id(p): eng.run(q, p, "baseline") for p in (pa, pb)}
    for p in (pa, pb, pa, pb, pb):
        eng.submit(q, p, "baseline")
        eng.sync()
        assert np.array_equal(eng.host_ids.numpy(), want[id(p)])
    for _ in range(4):  # back to back without host synchronisation: the last batch's lists land
        eng.submit(q, pa, "baseline")
    eng.submit(q, pb, "baseline")
    eng.sync()
    assert np.array_equal(eng.host_ids.numpy(), want[id(pb)])
