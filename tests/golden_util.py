"""Load the golden fixtures (tests/golden/*.npz, made by make_golden.py from
the reference) into this package's types."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2507_17094_b200.data import Dataset
from paper_2507_17094_b200.graphs import Index, ShardPack
from paper_2507_17094_b200.search import GhostContext, SearchParams, ShardContext

GOLDEN = Path(__file__).resolve().parent / "golden"
STAT_FIELDS = ("iterations", "ghost_iterations", "distance_computations", "total_visits",
               "inserted", "retained", "dgs_skipped", "converged")

ARMS_SMALL = []
for _sel, _dr in (("full", 0.0), ("direction", 0.5), ("random", 0.5)):
    for _ghost in (False, True):
        for _sm in ("neighbors", "mixed"):
            ARMS_SMALL.append(dict(selection=_sel, discard_ratio=_dr, ghost_enabled=_ghost,
                                   seed_mode=_sm))
SMALL_BASE = dict(k=10, l=32, m=32, r=4, max_iter=24, seed=17, cooldown_ratio=0.3,
                  ghost_max_iter=6)
EXTRA_SMALL = [dict(k=10, l=32, m=32, r=4, max_iter=3, seed=3),
               dict(k=5, l=16, m=8, r=2, max_iter=30, seed=4, buffer_cap=10),
               dict(k=10, l=64, m=100, r=8, max_iter=40, seed=5, selection="direction",
                    discard_ratio=0.25, cooldown_ratio=0.5, ghost_enabled=True, ghost_max_iter=3)]
ARMS_SIFT = [dict(),
             dict(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3),
             dict(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3,
                  ghost_enabled=True, ghost_max_iter=8)]
SIFT_BASE = dict(k=10, l=64, m=64, r=8, max_iter=64, seed=0)


def small_cases():
    """(name, params, prefix) for every golden run in small.npz."""
    out = []
    for i, arm in enumerate(ARMS_SMALL):
        for mode in ("baseline", "pipelined"):
            out.append((f"arm{i:02d}-{mode}", SearchParams(**SMALL_BASE, **arm), mode,
                        f"arm{i:02d}_{mode}_"))
    for i, kw in enumerate(EXTRA_SMALL):
        for mode in ("baseline", "pipelined"):
            out.append((f"extra{i}-{mode}", SearchParams(**kw), mode, f"extra{i}_{mode}_"))
    return out


def sift_cases():
    out = []
    for i, arm in enumerate(ARMS_SIFT):
        for mode in ("baseline", "pipelined"):
            out.append((f"sift{i}-{mode}", SearchParams(**SIFT_BASE, **arm), mode,
                        f"arm{i:02d}_{mode}_"))
    return out


def pack_sign_bits(bits: np.ndarray) -> np.ndarray:
    """direction.py:28-38 (little-endian bit order inside uint32 words)."""
    d = bits.shape[-1]
    w = (d + 31) // 32
    pad = w * 32 - d
    if pad:
        bits = np.concatenate([bits, np.zeros(bits.shape[:-1] + (pad,), bool)], axis=-1)
    return np.ascontiguousarray(np.packbits(bits, axis=-1, bitorder="little")).view("<u4")


def direction_table(vectors: np.ndarray, adj: np.ndarray) -> np.ndarray:
    """graphs.py:177-186 build_direction_table."""
    return pack_sign_bits(vectors[adj] >= vectors[:, None, :])


def load(name: str):
    """-> (npz, base Dataset, queries (Q,d) f32, Index, [ShardContext])."""
    z = np.load(GOLDEN / f"{name}.npz")
    base = z["base"]
    n_shards = int(z["n_shards"])
    packs, ctxs = [], []
    for s in range(n_shards):
        g = z[f"s{s}_global_ids"]
        adj = z[f"s{s}_adj"]
        vec = np.ascontiguousarray(base[g])
        if f"s{s}_direction" in z:
            direction = z[f"s{s}_direction"]
        else:
            direction = direction_table(vec, adj)
            assert np.uint64(direction.astype(np.uint64).sum()) == z[f"s{s}_direction_sum"]
            assert np.uint32(np.bitwise_xor.reduce(direction.ravel())) == z[f"s{s}_direction_xor"]
        inter = z[f"s{s}_inter_map"] if f"s{s}_inter_map" in z else None
        gids = z[f"s{s}_ghost_ids"] if f"s{s}_ghost_ids" in z else None
        gadj = z[f"s{s}_ghost_adj"] if f"s{s}_ghost_adj" in z else None
        packs.append(ShardPack(g, adj, inter, gids, gadj, direction))
        ghost = None if gids is None else GhostContext(vectors=vec[gids], adj=gadj, parent_ids=gids)
        ctxs.append(ShardContext(vectors=vec, adj=adj, global_ids=g, direction=direction,
                                 inter_map=inter, ghost=ghost))
    index = Index(d=base.shape[1], n_total=base.shape[0], shards=packs)
    return z, Dataset(base), np.ascontiguousarray(z["queries"]), index, ctxs


def expected(z, prefix: str) -> dict:
    out = dict(final_ids=z[prefix + "final_ids"], final_dists=z[prefix + "final_dists"],
               shard_ids=z[prefix + "shard_ids"], shard_dists=z[prefix + "shard_dists"],
               comm=z[prefix + "comm"])
    for f in STAT_FIELDS:
        out[f] = z[prefix + "stat_" + f]
    return out


def assert_run_equal(got: dict, want: dict, what: str) -> None:
    """Every array of a PipelineResult-like dict equal (bit-exact)."""
    for key in ("final_ids", "final_dists", "shard_ids", "shard_dists"):
        a, b = np.asarray(got[key]), np.asarray(want[key])
        assert a.shape == b.shape, (what, key, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{what}: {key} differs at {bad.tolist()}")
    assert np.array_equal(got["comm"], want["comm"]), (what, "comm")
    for f in STAT_FIELDS:
        a, b = np.asarray(got[f]), np.asarray(want[f])
        if not np.array_equal(a.astype(np.int64), b.astype(np.int64)):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{what}: stat {f} differs at {bad.tolist()}")


def result_dict(res) -> dict:
    """PipelineResult -> dict in the golden layout."""
    out = dict(final_ids=res.final_ids, final_dists=res.final_dists, shard_ids=res.shard_ids,
               shard_dists=res.shard_dists, comm=res.comm_stage_bytes)
    for f in STAT_FIELDS:
        out[f] = np.stack([getattr(st, f) for st in res.stages])
    return out


def oracle_dict(res: dict) -> dict:
    out = dict(final_ids=res["final_ids"], final_dists=res["final_dists"],
               shard_ids=res["shard_ids"], shard_dists=res["shard_dists"],
               comm=res["comm_stage_bytes"])
    for f in STAT_FIELDS:
        out[f] = np.stack([st[f] for st in res["stages"]])
    return out


def assert_run_equal_lossy(got: dict, want: dict, what: str) -> None:
    """Lossy visited cache (tuning flag 2): every array and counter equal to
    the exact run except distance_computations, which may only grow (forgotten
    nodes are re-scored and then dropped by the merge)."""
    dc = "distance_computations"
    assert np.all(np.asarray(got[dc]) >= np.asarray(want[dc])), (what, "distance_computations shrank")
    g = dict(got)
    g[dc] = want[dc]
    assert_run_equal(g, want, what)
