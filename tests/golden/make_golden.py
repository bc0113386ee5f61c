"""Generate the golden fixtures under tests/golden/ from the reference itself.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference package (shardann 0.1.0, pure Python/numpy) is imported from
/root/reference/pkg/src; every output here is produced by ITS code, so the
fixtures pin both the CPU oracle (oracle/) and the CUDA path.  Nothing at test
time reads /root/reference.

Fixtures:
* rng.npz      derive_seed / PCG64 seeding / Generator.choice / permutation
               (rng.py:26-44, search.py:222, direction.py:105)
* l2.npz       squared_l2 outputs at d in {1,2,7,16,32,96,128,200,960} (data.py:70-79)
* small.npz    conftest.py small_data + small_index (4 shards, d=16) and the
               outputs of run_sharded_baseline / run_pipelined for 24 arms
               (pipeline.py:270-350): ids, dists, every StageStats array, comm
* sift128.npz  a d=128 / j=32 / 2-shard index (3000 points, 64 queries) plus the
               outputs of 6 arms (SIFT-shaped rows at desk scale)
* search.npz   single-search cases mirroring tests/test_search.py of the reference
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import shardann as sa  # noqa: E402
from shardann.rng import TAG_GHOST_SEARCH, TAG_SEARCH, derive_seed, stream  # noqa: E402

OUT = Path(__file__).resolve().parent
STAT_FIELDS = ("iterations", "ghost_iterations", "distance_computations", "total_visits",
               "inserted", "retained", "dgs_skipped", "converged")


def _index_arrays(prefix, index, base):
    out = {}
    for s, p in enumerate(index.shards):
        out[f"{prefix}s{s}_global_ids"] = p.global_ids
        out[f"{prefix}s{s}_adj"] = p.adj
        if p.inter_map is not None:
            out[f"{prefix}s{s}_inter_map"] = p.inter_map
        if p.ghost_ids is not None:
            out[f"{prefix}s{s}_ghost_ids"] = p.ghost_ids
            out[f"{prefix}s{s}_ghost_adj"] = p.ghost_adj
        if p.direction is not None:
            out[f"{prefix}s{s}_direction"] = p.direction
    return out


def _result_arrays(prefix, res):
    out = {f"{prefix}final_ids": res.final_ids, f"{prefix}final_dists": res.final_dists,
           f"{prefix}shard_ids": res.shard_ids, f"{prefix}shard_dists": res.shard_dists,
           f"{prefix}comm": res.comm_stage_bytes}
    for f in STAT_FIELDS:
        out[f"{prefix}stat_{f}"] = np.stack([getattr(st, f) for st in res.stages])
    return out


ARMS_SMALL = []
for sel, dr in (("full", 0.0), ("direction", 0.5), ("random", 0.5)):
    for ghost in (False, True):
        for sm in ("neighbors", "mixed"):
            ARMS_SMALL.append(dict(selection=sel, discard_ratio=dr, ghost_enabled=ghost,
                                   seed_mode=sm))


def arm_name(i, mode):
    return f"arm{i:02d}_{mode}_"


def make_rng():
    rs = np.random.default_rng(1)
    seeds = [0, 1, 5, 2**32 - 1, 2**32, 2**63 + 5] + [derive_seed(0, 4, q, s) for q in range(5) for s in range(3)]
    states = []
    for sd in seeds:
        st = np.random.PCG64(sd).state
        states.append([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                       st["state"]["inc"] >> 64, st["state"]["inc"] & (2**64 - 1)])
    ds_parts = np.array([[s, t, q, g] for s in (0, 7, 17, 2**40) for t in (4, 5) for q in (0, 1, 999)
                         for g in (0, 3)], dtype=np.uint64)
    ds_out = np.array([derive_seed(int(a), int(b), int(c), int(d)) for a, b, c, d in ds_parts],
                      dtype=np.uint64)
    cases, outs = [], []
    for _ in range(200):
        pop = int(rs.choice([25, 100, 1000, 9999, 10001, 12000, 50000, 12_500_000]))
        size = int(rs.integers(1, min(pop, 300) + 1))
        sd = int(rs.integers(0, 2**63))
        g = np.random.Generator(np.random.PCG64(sd))
        o = g.choice(pop, size, replace=False)
        st = g.bit_generator.state
        cases.append([sd, pop, size, st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                      st["has_uint32"], st["uinteger"]])
        outs.append(np.pad(o, (0, 300 - size), constant_values=-1))
    perm_cases, perm_outs = [], []
    for _ in range(50):
        n = int(rs.integers(1, 65))
        sd = int(rs.integers(0, 2**63))
        g = np.random.Generator(np.random.PCG64(sd))
        perm_cases.append([sd, n])
        perm_outs.append(np.pad(g.permutation(n), (0, 64 - n), constant_values=-1))
    np.savez_compressed(
        OUT / "rng.npz", seeds=np.array(seeds, dtype=np.uint64),
        states=np.array(states, dtype=np.uint64), ds_parts=ds_parts, ds_out=ds_out,
        choice_cases=np.array(cases, dtype=np.uint64), choice_out=np.array(outs, dtype=np.int64),
        perm_cases=np.array(perm_cases, dtype=np.uint64), perm_out=np.array(perm_outs, np.int64))


def make_l2():
    rs = np.random.default_rng(2)
    out = {}
    for d in (1, 2, 7, 16, 32, 96, 128, 200, 960):
        x = (rs.standard_normal((40, d)) * 3).astype(np.float32)
        q = (rs.standard_normal(d) * 3).astype(np.float32)
        out[f"x{d}"] = x
        out[f"q{d}"] = q
        out[f"sq{d}"] = sa.squared_l2(x, q)
    np.savez_compressed(OUT / "l2.npz", **out)


def make_small():
    full = sa.gen_synthetic(4100, 16, 32, 0.2, seed=99)
    base = sa.Dataset(full.data[:4000])
    queries = sa.Dataset(full.data[4000:])
    index, _ = sa.build_index(base, 4, 16, seed=5, rho=0.05, ghost_degree=8)
    ctxs = sa.build_contexts(index, base)
    out = dict(base=base.data, queries=queries.data, n_shards=np.int32(4))
    out.update(_index_arrays("", index, base))
    truth = sa.exact_knn_batch(base, queries, 10)
    out["truth_ids"] = np.stack([t.ids for t in truth])
    out["truth_dists"] = np.stack([t.dists for t in truth])
    for i, arm in enumerate(ARMS_SMALL):
        params = sa.SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17, cooldown_ratio=0.3,
                                 ghost_max_iter=6, **arm)
        for mode, runner in (("baseline", sa.run_sharded_baseline), ("pipelined", sa.run_pipelined)):
            out.update(_result_arrays(arm_name(i, mode), runner(queries, index, base, params,
                                                                 contexts=ctxs)))
    # budget-limited (non-converged) and buffer-capped variants
    extra = [dict(k=10, l=32, m=32, r=4, max_iter=3, seed=3),
             dict(k=5, l=16, m=8, r=2, max_iter=30, seed=4, buffer_cap=10),
             dict(k=10, l=64, m=100, r=8, max_iter=40, seed=5, selection="direction",
                  discard_ratio=0.25, cooldown_ratio=0.5, ghost_enabled=True, ghost_max_iter=3)]
    for i, kw in enumerate(extra):
        params = sa.SearchParams(**kw)
        for mode, runner in (("baseline", sa.run_sharded_baseline), ("pipelined", sa.run_pipelined)):
            out.update(_result_arrays(f"extra{i}_{mode}_", runner(queries, index, base, params,
                                                                   contexts=ctxs)))
    np.savez_compressed(OUT / "small.npz", **out)


ARMS_SIFT = [
    dict(),
    dict(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3),
    dict(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3, ghost_enabled=True,
         ghost_max_iter=8),
]


def make_sift128():
    full = sa.gen_synthetic(3064, 128, 96, 0.08, seed=0)
    base = sa.Dataset(full.data[:3000])
    queries = sa.Dataset(full.data[3000:])
    index, _ = sa.build_index(base, 2, 32, seed=0, rho=0.02, ghost_degree=16)
    ctxs = sa.build_contexts(index, base)
    out = dict(base=base.data, queries=queries.data, n_shards=np.int32(2))
    arrs = _index_arrays("", index, base)
    # direction tables are re-derived at load (direction.py:28-38 on vectors/adj);
    # keep a checksum so the loader proves the rebuild is exact
    for s in range(2):
        d = arrs.pop(f"s{s}_direction")
        out[f"s{s}_direction_sum"] = np.uint64(d.astype(np.uint64).sum())
        out[f"s{s}_direction_xor"] = np.uint32(np.bitwise_xor.reduce(d.ravel()))
    out.update(arrs)
    for i, arm in enumerate(ARMS_SIFT):
        params = sa.SearchParams(k=10, l=64, m=64, r=8, max_iter=64, seed=0, **arm)
        for mode, runner in (("baseline", sa.run_sharded_baseline), ("pipelined", sa.run_pipelined)):
            out.update(_result_arrays(arm_name(i, mode), runner(queries, index, base, params,
                                                                 contexts=ctxs)))
    np.savez_compressed(OUT / "sift128.npz", **out)


def _line_context(n=10, j=4):
    vectors = np.arange(n, dtype=np.float32)[:, None]
    adj = np.empty((n, j), dtype=np.int32)
    for u in range(n):
        others = sorted((abs(v - u), v) for v in range(n) if v != u)
        adj[u] = [v for _, v in others[:j]]
    return sa.ShardContext(vectors=vectors, adj=adj, global_ids=np.arange(n, dtype=np.int32))


def make_search():
    """Single-search cases (search.py:269) mirroring the reference's test_search.py."""
    out = {}
    # complete graph == exact kNN (test_search.py:105-115)
    full = sa.gen_synthetic(64, 8, 4, 0.3, seed=3)
    adj = sa.build_knn_graph(full.data, 63)
    out["complete_vectors"] = full.data
    out["complete_adj"] = adj
    params = sa.SearchParams(k=10, l=16, m=8, r=2, max_iter=20, seed=5)
    ids, dists = [], []
    ctx = sa.ShardContext(vectors=full.data, adj=adj, global_ids=full.ids)
    for qi in range(10):
        q = full.data[qi] + 0.01
        res = sa.search(q, ctx, params, seeds=(0,), rng=stream(5, TAG_SEARCH, qi, 0))
        ids.append(res.ids)
        dists.append(res.dists)
    out["complete_ids"] = np.stack(ids)
    out["complete_dists"] = np.stack(dists)
    # buffer cap visit order (test_search.py:197-205)
    lc = _line_context(n=10, j=8)
    out["line_adj"] = lc.adj
    params = sa.SearchParams(k=1, l=4, m=1, r=1, max_iter=2, seed=0, buffer_cap=5, log_visits=True)
    res = sa.search(np.zeros(1, np.float32), lc, params, seeds=(9,), rng=stream(0, TAG_SEARCH, 0, 0))
    out["line_visited"] = res.visited_ids
    out["line_total_visits"] = np.int64(res.counters.total_visits)
    # log_visits on a random graph + explicit rng state round trip
    full = sa.gen_synthetic(800, 8, 8, 0.2, seed=8)
    adj = sa.build_knn_graph(full.data, 8)
    out["visit_vectors"] = full.data
    out["visit_adj"] = adj
    params = sa.SearchParams(k=5, l=16, m=16, r=4, max_iter=12, seed=2, log_visits=True)
    g = stream(2, TAG_SEARCH, 3, 0)
    res = sa.search(full.data[3], sa.ShardContext(vectors=full.data, adj=adj, global_ids=full.ids),
                    params, rng=g)
    out["visit_log"] = res.visited_ids
    out["visit_ids"] = res.ids
    out["visit_dists"] = res.dists
    c = res.counters
    out["visit_counters"] = np.array([c.iterations, c.distance_computations, c.total_visits,
                                      c.nodes_expanded, c.dgs_skipped, c.inserted_total], np.int64)
    st = g.bit_generator.state
    out["visit_rng_after"] = np.array([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                                       st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    np.savez_compressed(OUT / "search.npz", **out)


if __name__ == "__main__":
    make_rng()
    make_l2()
    make_search()
    make_small()
    make_sift128()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
