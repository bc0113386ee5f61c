"""Parity of the CUDA path (through the C ABI) with the reference.

* golden fixtures produced by the reference itself (tests/golden/): every
  array of every PipelineResult bit-equal, every counter equal;
* the CPU oracle (pinned to the same goldens) at sizes/dims the fixtures do
  not cover (d = 96 / 128 / 200 / 960, 2-4 shards, thousands of queries).
"""

from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2507_17094_b200 as pw
from golden_util import (GOLDEN, assert_run_equal, assert_run_equal_lossy, expected, load, oracle_dict, result_dict,
                         sift_cases, small_cases)
from paper_2507_17094_b200.rng import TAG_SEARCH, stream
from paper_2507_17094_b200.search import SearchParams, ShardContext

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small():
    z, base, queries, index, ctxs = load("small")
    return z, base, pw.Dataset(queries), index, pw.build_contexts(index, base)


@pytest.fixture(scope="module")
def sift():
    z, base, queries, index, ctxs = load("sift128")
    return z, base, pw.Dataset(queries), index, pw.build_contexts(index, base)


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c[0])
def test_small_golden(small, case):
    name, params, mode, prefix = case
    z, base, queries, index, ctxs = small
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(queries, index, base, params, contexts=ctxs))
    assert_run_equal(got, expected(z, prefix), name)


@pytest.mark.parametrize("case", sift_cases(), ids=lambda c: c[0])
def test_sift128_golden(sift, case):
    name, params, mode, prefix = case
    z, base, queries, index, ctxs = sift
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(queries, index, base, params, contexts=ctxs))
    assert_run_equal(got, expected(z, prefix), name)


def test_build_contexts_from_index(small):
    z, base, queries, index, _ = small
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17, cooldown_ratio=0.3,
                          ghost_max_iter=6)
    got = result_dict(pw.run_pipelined(queries, index, base, params))
    assert_run_equal(got, expected(z, "arm00_pipelined_"), "contexts=None")


@pytest.mark.parametrize("d", [1, 2, 7, 16, 32, 96, 128, 200, 960])
def test_squared_l2_primitive_golden(d):
    import torch

    z = np.load(GOLDEN / "l2.npz")
    x, q = z[f"x{d}"], z[f"q{d}"]
    ctx = ShardContext(vectors=x, adj=np.zeros((x.shape[0], 0), np.int32),
                       global_ids=np.arange(x.shape[0], dtype=np.int32))
    dev = pw.device_shard(ctx)
    lib = pw._abi.load()
    ids = torch.arange(x.shape[0], dtype=torch.int32, device="cuda")
    tq = torch.from_numpy(q).cuda()
    out = torch.empty(x.shape[0], dtype=torch.float32, device="cuda")
    pw._abi.check(lib.pw_squared_l2_rows(dev.handle, ids.data_ptr(), x.shape[0], tq.data_ptr(),
                                         out.data_ptr(), None))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), z[f"sq{d}"])


def _ctx(vectors, adj):
    return ShardContext(vectors=vectors, adj=adj, global_ids=np.arange(vectors.shape[0], dtype=np.int32))


def test_search_complete_graph_exact():
    """reference tests/test_search.py:105-115 (ids AND dists bit-equal)."""
    z = np.load(GOLDEN / "search.npz")
    ctx = _ctx(z["complete_vectors"], z["complete_adj"])
    params = SearchParams(k=10, l=16, m=8, r=2, max_iter=20, seed=5)
    for qi in range(10):
        q = ctx.vectors[qi] + np.float32(0.01)
        res = pw.search(q, ctx, params, seeds=(0,), rng=stream(5, TAG_SEARCH, qi, 0))
        assert res.ids.tolist() == z["complete_ids"][qi].tolist()
        assert np.array_equal(res.dists, z["complete_dists"][qi])
        assert res.converged


def test_search_buffer_cap_visit_order():
    """reference tests/test_search.py:197-205."""
    z = np.load(GOLDEN / "search.npz")
    ctx = _ctx(np.arange(10, dtype=np.float32)[:, None], z["line_adj"])
    params = SearchParams(k=1, l=4, m=1, r=1, max_iter=2, seed=0, buffer_cap=5, log_visits=True)
    res = pw.search(np.zeros(1, np.float32), ctx, params, seeds=(9,), rng=stream(0, TAG_SEARCH, 0, 0))
    assert res.visited_ids.tolist() == z["line_visited"].tolist()
    assert res.counters.total_visits == int(z["line_total_visits"])


def test_search_visit_log_counters_and_rng_state():
    """log_visits order, all counters, and the caller's Generator advanced like numpy."""
    z = np.load(GOLDEN / "search.npz")
    ctx = _ctx(z["visit_vectors"], z["visit_adj"])
    params = SearchParams(k=5, l=16, m=16, r=4, max_iter=12, seed=2, log_visits=True)
    g = stream(2, TAG_SEARCH, 3, 0)
    res = pw.search(ctx.vectors[3], ctx, params, rng=g)
    assert res.visited_ids.tolist() == z["visit_log"].tolist()
    assert res.ids.tolist() == z["visit_ids"].tolist()
    assert np.array_equal(res.dists, z["visit_dists"])
    c = res.counters
    assert [c.iterations, c.distance_computations, c.total_visits, c.nodes_expanded,
            c.dgs_skipped, c.inserted_total] == z["visit_counters"].tolist()
    st = g.bit_generator.state
    after = z["visit_rng_after"]
    assert st["state"]["state"] == (int(after[0]) << 64) | int(after[1])
    assert st["has_uint32"] == int(after[2]) and st["uinteger"] == int(after[3])


def test_single_node_graph():
    """reference tests/test_search.py:118-128 (degree-0 graph)."""
    ctx = ShardContext(vectors=np.array([[1.0, 2.0]], dtype=np.float32),
                       adj=np.empty((1, 0), dtype=np.int32), global_ids=np.array([7], dtype=np.int32))
    params = SearchParams(k=1, l=4, m=4, r=1, max_iter=8, seed=0)
    res = pw.search(np.array([1.0, 0.0]), ctx, params, rng=stream(0, TAG_SEARCH, 0, 0))
    assert res.ids.tolist() == [7]
    assert res.dists[0] == pytest.approx(2.0)
    assert res.converged


def test_search_matches_oracle_all_selections(small):
    z, base, queries, index, ctxs = small
    ctx = ctxs[1]
    for sel, dr in (("full", 0.0), ("direction", 0.5), ("random", 0.5)):
        params = SearchParams(k=10, l=32, m=32, r=4, max_iter=16, seed=9, selection=sel,
                              discard_ratio=dr, cooldown_ratio=0.25, log_visits=True)
        for qi in range(0, 100, 9):
            q = queries.data[qi]
            g = stream(9, TAG_SEARCH, qi, 1)
            res = pw.search(q, ctx, params, rng=g)
            want, st = oracle.search(q, ctx, params, rng_state=oracle.pcg64_state(
                pw.rng.derive_seed(9, TAG_SEARCH, qi, 1)))
            assert res.ids.tolist() == want["ids"].tolist()
            assert np.array_equal(res.dists, want["dists"])
            assert res.visited_ids.tolist() == want["visited_ids"].tolist()
            assert res.counters.__dict__ == want["counters"]
            assert g.bit_generator.state["state"] == st["state"]


def test_ghost_stage_matches_oracle(small):
    z, base, queries, index, ctxs = small
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17, ghost_enabled=True,
                          ghost_max_iter=6)
    for s, ctx in enumerate(ctxs):
        for qi in range(0, 100, 13):
            g = stream(17, 5, qi, s)
            entry, counters = pw.run_ghost_stage(queries.data[qi], ctx, params, rng=g)
            e2, c2, _ = oracle.ghost_stage(queries.data[qi], ctx, params, rng_state=oracle.pcg64_state(
                pw.rng.derive_seed(17, 5, qi, s)))
            assert entry == e2
            assert counters.iterations == c2["iterations"]
            assert counters.distance_computations == c2["distance_computations"]


def test_ghost_stage_identity_with_full_sample(small):
    """reference tests/test_pipeline.py:137-159 with ghost graph == main graph."""
    z, base, queries, index, ctxs = small
    v = ctxs[0].vectors[:500]
    from index_util import knn_graph
    adj = knn_graph(v, 8)
    ids = np.arange(500, dtype=np.int32)
    ctx = ShardContext(vectors=v, adj=adj, global_ids=ids,
                       ghost=pw.GhostContext(vectors=v, adj=adj, parent_ids=ids))
    params = SearchParams(k=1, l=16, m=16, r=4, max_iter=6, seed=5, ghost_enabled=True,
                          ghost_max_iter=6)
    for qi in range(5):
        q = queries.data[qi]
        entry, counters = pw.run_ghost_stage(q, ctx, params, rng=stream(5, TAG_SEARCH, qi, 0))
        res = pw.search(q, ctx, params.with_(k=1, ghost_enabled=False),
                        rng=stream(5, TAG_SEARCH, qi, 0), query_id=qi)
        assert entry == res.local_ids[0]
        assert counters.iterations <= params.ghost_max_iter


def test_reduce_topk_goldens():
    """reference tests/test_pipeline.py:48-69."""
    ids, dists = pw.reduce_topk(np.array([5, 9, 1]), np.array([0.5, 0.1, 0.9], np.float32), 2)
    assert ids.tolist() == [9, 5]
    ids, dists = pw.reduce_topk(np.array([3, 2, -1, 7]), np.array([0.5, 0.5, np.inf, 0.25], np.float32), 3)
    assert ids.tolist() == [7, 2, 3]
    with pytest.raises(ValueError, match="empty"):
        pw.reduce_topk(np.array([-1, -1]), np.array([np.inf, np.inf], np.float32), 2)


def test_validation_errors(small):
    z, base, queries, index, ctxs = small
    params = SearchParams(k=1, l=4, m=4, r=1, max_iter=4, seed=0)
    line = _ctx(np.arange(10, dtype=np.float32)[:, None], np.zeros((10, 2), np.int32))
    with pytest.raises(ValueError, match="seed"):
        pw.search(np.zeros(1, np.float32), line, params, seeds=(99,), rng=stream(0, 4, 0, 0))
    with pytest.raises(ValueError, match="does not match"):
        pw.search(np.zeros(3, np.float32), line, params, rng=stream(0, 4, 0, 0))
    with pytest.raises(ValueError, match="direction table"):
        pw.search(np.zeros(1, np.float32), line, params.with_(selection="direction", discard_ratio=0.5),
                  rng=stream(0, 4, 0, 0))
    with pytest.raises(ValueError, match="ghost"):
        pw.run_ghost_stage(np.zeros(1, np.float32), line, params.with_(ghost_enabled=True),
                           rng=stream(0, 4, 0, 0))
    stripped = pw.Index(d=index.d, n_total=index.n_total,
                        shards=[pw.ShardPack(p.global_ids, p.adj, None, None, None, None)
                                for p in index.shards])
    with pytest.raises(ValueError, match="inter-shard"):
        pw.run_pipelined(queries, stripped, base, params)
    with pytest.raises(ValueError, match="does not match"):
        pw.build_contexts(index, pw.Dataset(np.zeros((base.n, base.d + 1), np.float32)))


@pytest.fixture(scope="module")
def synth():
    from index_util import clustered, make_contexts
    out = {}
    for d, n, nq, shards, j in ((96, 24000, 600, 2, 32), (128, 12000, 300, 3, 32),
                                (200, 6000, 200, 2, 24), (960, 3000, 64, 2, 32)):
        x = clustered(n + nq, d, 512, 0.08, seed=d)
        out[d] = (np.ascontiguousarray(x[n:]), make_contexts(x[:n], shards, j, seed=d))
    return out


SYNTH_ARMS = [
    dict(k=10, l=64, m=64, r=8, max_iter=64, seed=1),
    dict(k=10, l=128, m=64, r=8, max_iter=64, seed=2, selection="direction", discard_ratio=0.5,
         cooldown_ratio=0.3, ghost_enabled=True, ghost_max_iter=8),
    dict(k=10, l=96, m=64, r=4, max_iter=10, seed=3, selection="random", discard_ratio=0.5,
         seed_mode="mixed", ghost_enabled=True),
    dict(k=16, l=256, m=128, r=16, max_iter=64, seed=4),
]


@pytest.mark.parametrize("d", [96, 128, 200, 960])
@pytest.mark.parametrize("arm", range(len(SYNTH_ARMS)))
@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
def test_synthetic_matches_oracle(synth, d, arm, mode):
    queries, ctxs = synth[d]
    params = SearchParams(**SYNTH_ARMS[arm])
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(pw.Dataset(queries), None, None, params, contexts=ctxs))
    want = oracle_dict(oracle.run(queries, ctxs, params, mode))
    assert_run_equal(got, want, f"d={d} arm={arm} {mode}")


def test_visited_spill_to_global_table(synth):
    """Tiny shared-memory visited table forces the exact global spill path."""
    queries, ctxs = synth[96]
    params = SearchParams(**SYNTH_ARMS[3])
    got = result_dict(pw.run_sharded_baseline(pw.Dataset(queries), None, None, params, contexts=ctxs,
                                              tuning={"visited_slots": 256}))
    want = oracle_dict(oracle.run(queries, ctxs, params, "baseline"))
    assert_run_equal(got, want, "spill")


LOSSY = {"flags": 2}


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c[0])
@pytest.mark.parametrize("slots", [8192, 256])
def test_small_golden_lossy_visited(small, case, slots):
    """Lossy visited cache: ids, distances and every counter but
    distance_computations identical to the reference; 256 slots (the
    minimum) forces heavy
    forgetting, so re-scored queued nodes must be dropped by the merge."""
    name, params, mode, prefix = case
    if params.log_visits:
        pytest.skip("the visit log needs the exact set (lossy is ignored)")
    z, base, queries, index, ctxs = small
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(queries, index, base, params, contexts=ctxs,
                             tuning=dict(LOSSY, visited_slots=slots)))
    assert_run_equal_lossy(got, expected(z, prefix), f"{name} lossy {slots}")


@pytest.mark.parametrize("d", [96, 128, 200, 960])
@pytest.mark.parametrize("arm", range(len(SYNTH_ARMS)))
@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
@pytest.mark.parametrize("slots", [8192, 256])
def test_synthetic_lossy_visited_matches_oracle(synth, d, arm, mode, slots):
    queries, ctxs = synth[d]
    params = SearchParams(**SYNTH_ARMS[arm])
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(pw.Dataset(queries), None, None, params, contexts=ctxs,
                             tuning=dict(LOSSY, visited_slots=slots)))
    want = oracle_dict(oracle.run(queries, ctxs, params, mode))
    assert_run_equal_lossy(got, want, f"d={d} arm={arm} {mode} lossy {slots}")


def test_lossy_visited_ids_beyond_24_bits():
    """The lossy cache's words hold epoch8 << 24 | the low bits of a bijective
    hash, so shards of >= 2^24 nodes keep exact hits (a false hit would skip
    a node and change the result).  17M points on a line (d = 1) with a
    small-world graph; queries sit beyond id 2^24."""
    import torch
    n = (1 << 24) + 600_000
    rs = np.random.default_rng(24)
    x = np.arange(n, dtype=np.float32)[:, None] * np.float32(1.0 / 64)
    off = np.array([-3, -2, -1, 1, 2, 3], np.int64)
    idx = np.arange(n, dtype=np.int64)[:, None]
    adj = np.empty((n, 8), np.int32)
    adj[:, :6] = np.clip(idx + off, 0, n - 1)
    adj[:, 6:] = rs.integers(0, n, (n, 2))  # long-range links
    ctx = ShardContext(vectors=x, adj=adj, global_ids=np.arange(n, dtype=np.int32))
    q = (np.float32((1 << 24) + 1000) + rs.random((64, 1), dtype=np.float32) * 500_000) / np.float32(64)
    params = SearchParams(k=10, l=48, m=48, r=4, max_iter=48, seed=7)
    want = oracle_dict(oracle.run(q, [ctx], params, "baseline"))
    assert (want["final_ids"] >= (1 << 24)).mean() > 0.5
    for slots in (4096, 256):
        got = result_dict(pw.run_sharded_baseline(pw.Dataset(q), None, None, params, contexts=[ctx],
                                                  tuning=dict(LOSSY, visited_slots=slots)))
        assert_run_equal_lossy(got, want, f"ids >= 2^24 lossy {slots}")
    del ctx
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
@pytest.mark.parametrize("m,seed_mode", [(300, "neighbors"), (300, "mixed"), (1000, "mixed")])
def test_initial_batch_choice_tail_shuffle(synth, mode, m, seed_mode):
    """numpy Generator.choice(pop, m, replace=False) takes its tail-shuffle
    branch when pop > 10000 and m > pop / 50 (the oracle is pinned to that
    branch in rng.npz): 12000-node shards with m = 300 / 1000 random seeds
    (search.py:222), with and without forwarded entries ahead of them."""
    queries, ctxs = synth[96]
    assert all(c.vectors.shape[0] > 10000 and m > c.vectors.shape[0] // 50 for c in ctxs)
    params = SearchParams(k=10, l=64, m=m, r=8, max_iter=12, seed=11, seed_mode=seed_mode)
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(pw.Dataset(queries[:200]), None, None, params, contexts=ctxs))
    want = oracle_dict(oracle.run(queries[:200], ctxs, params, mode))
    assert_run_equal(got, want, f"choice tail m={m} {seed_mode} {mode}")


@pytest.mark.parametrize("d", [96, 128, 200, 960])
@pytest.mark.parametrize("arm", range(len(SYNTH_ARMS)))
@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
@pytest.mark.parametrize("flags", [8, 10])
def test_tma_gather4_rows_match_oracle(synth, d, arm, mode, flags):
    """Scoring rows staged by TMA tile::gather4 (tuning flag 8; d = 960 rows
    do not fit one box and keep the cp.async path): same results."""
    queries, ctxs = synth[d]
    params = SearchParams(**SYNTH_ARMS[arm])
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(pw.Dataset(queries), None, None, params, contexts=ctxs, tuning={"flags": flags}))
    want = oracle_dict(oracle.run(queries, ctxs, params, mode))
    (assert_run_equal_lossy if flags & 2 else assert_run_equal)(got, want, f"tma d={d} arm={arm} {mode}")


@pytest.mark.parametrize("pinned", [False, True])
def test_pw_run_overlapped_upload(synth, pinned):
    """pw_run uploads the queries in growing chunks (256, 512, 1024, ... rows)
    on a copy stream while K1 runs, each chunk released by a flag K1 polls:
    1537 queries (a partial last chunk), page-locked or pageable, lossy (FAST kernel) and exact,
    repeated calls (epoch tags) -- every result equal to the oracle."""
    import torch
    queries, ctxs = synth[96]
    q = np.concatenate([queries, queries, queries])[:1537]
    if pinned:
        qp = torch.empty(q.shape, dtype=torch.float32, pin_memory=True).numpy()
        qp[:] = q
        q = qp
    params = SearchParams(**SYNTH_ARMS[1])
    want = oracle_dict(oracle.run(np.ascontiguousarray(q), ctxs, params, "pipelined"))
    for tuning in (None, LOSSY, None):
        got = result_dict(pw.run_pipelined(pw.Dataset(q), None, None, params, contexts=ctxs, tuning=tuning))
        (assert_run_equal_lossy if tuning else assert_run_equal)(got, want, f"upload pinned={pinned} {tuning}")


@pytest.fixture(scope="module")
def one_shard():
    from index_util import clustered, make_contexts
    x = clustered(24000 + 2600, 96, 512, 0.08, seed=7)
    return np.ascontiguousarray(x[24000:]), make_contexts(x[:24000], 1, 32, seed=7)


@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
def test_pw_run_one_shard_chunked_upload(one_shard, mode):
    """One shard and several upload chunks (the bench's e2e shape): 2600
    queries (a partial fourth chunk), exact and lossy, repeated
    calls (epoch tags) and a smaller batch in between -- ids, distances and
    every counter equal to the oracle."""
    import torch
    queries, ctxs = one_shard
    qp = torch.empty(queries.shape, dtype=torch.float32, pin_memory=True).numpy()
    qp[:] = queries
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    params = SearchParams(**SYNTH_ARMS[1])
    want = oracle_dict(oracle.run(queries, ctxs, params, mode))
    want_small = oracle_dict(oracle.run(queries[:1100], ctxs, params, mode))
    for tuning in (None, LOSSY, None, LOSSY):
        got = result_dict(runner(pw.Dataset(qp), None, None, params, contexts=ctxs, tuning=tuning))
        (assert_run_equal_lossy if tuning else assert_run_equal)(got, want, f"one shard {mode} {tuning}")
        got = result_dict(runner(pw.Dataset(qp[:1100]), None, None, params, contexts=ctxs, tuning=tuning))
        (assert_run_equal_lossy if tuning else assert_run_equal)(got, want_small, f"one shard small {mode} {tuning}")


def test_pw_run_upload_with_blocking_launches(tmp_path):
    """CUDA_LAUNCH_BLOCKING=1 (as under a profiler's serialised replay: the
    launch returns only when K1 ends): the chunked upload must be fully
    enqueued before K1 is launched, or K1 waits for copies never issued."""
    import os
    import subprocess
    import sys
    script = tmp_path / "blocking.py"
    script.write_text(
        "import sys\n"
        f"sys.path[:0] = [{str(Path(__file__).parent)!r}, {str(Path(__file__).parent.parent)!r}]\n"
        "import numpy as np\n"
        "import paper_2507_17094_b200 as pw\n"
        "from index_util import clustered, make_contexts\n"
        "from paper_2507_17094_b200.search import SearchParams\n"
        "x = clustered(6000 + 1300, 32, 64, 0.08, seed=3)\n"
        "ctxs = make_contexts(x[:6000], 1, 16, seed=3)\n"
        "p = SearchParams(k=10, l=32, m=32, r=4, max_iter=16, seed=1)\n"
        "r = pw.run_pipelined(pw.Dataset(np.ascontiguousarray(x[6000:])), None, None, p, contexts=ctxs)\n"
        "print('ok', r.final_ids.shape)\n")
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    out = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok (1300, 10)" in out.stdout, out.stderr[-2000:]


def test_pw_run_result_block_and_separate_buffers(one_shard, synth):
    """pw_run's results are the same whether the six host buffers form the
    documented result block (one copy back) or are separate allocations (six
    copies): byte-equal arrays, one shard and a pipelined 2-shard run."""
    import ctypes as C

    from paper_2507_17094_b200 import _abi
    from paper_2507_17094_b200.pipeline import device_shard
    lib = _abi.load()
    params = SearchParams(**SYNTH_ARMS[1])
    for queries, ctxs in (one_shard, synth[96]):
        devs = [device_shard(c) for c in ctxs]
        n, q, k = len(devs), queries.shape[0], params.k
        handles = (C.c_void_p * n)(*[d.handle.value for d in devs])
        p, t = _abi.params_struct(params), _abi.tuning_struct(None)
        blk = _abi.result_block(q, n, k)
        sep = dict(shard_ids=np.empty((q, n, k), np.int32), shard_dists=np.empty((q, n, k), np.float32),
                   final_ids=np.empty((q, k), np.int32), final_dists=np.empty((q, k), np.float32),
                   s32=np.empty((n, 4, q), np.int32), s64=np.empty((n, 6, q), np.int64))
        for out in (blk, sep):
            comm = np.empty((n, n), np.int64)
            _abi.check(lib.pw_run(handles, n, C.byref(p), C.byref(t), queries.ctypes.data, q, 1,
                                  out["shard_ids"].ctypes.data, out["shard_dists"].ctypes.data,
                                  out["final_ids"].ctypes.data, out["final_dists"].ctypes.data,
                                  out["s32"].ctypes.data, out["s64"].ctypes.data, comm.ctypes.data))
        for key in sep:
            assert np.array_equal(blk[key].view(np.uint8), sep[key].view(np.uint8)), (n, key)
