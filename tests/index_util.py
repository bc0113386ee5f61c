"""Deterministic test-only index builder (numpy) for parity tests at sizes the
golden fixtures do not cover.  The graph need not equal the reference's
build_index: the CUDA path and the oracle search the SAME arrays."""

from __future__ import annotations

import numpy as np

from golden_util import direction_table
from paper_2507_17094_b200.search import GhostContext, ShardContext


def clustered(n: int, d: int, n_clusters: int, spread: float, seed: int) -> np.ndarray:
    rs = np.random.default_rng(seed)
    centers = rs.random((n_clusters, d), dtype=np.float32)
    noise = rs.standard_normal((n, d), dtype=np.float32) * np.float32(spread)
    return centers[np.arange(n) % n_clusters] + noise


def knn_graph(x: np.ndarray, j: int, exclude_self: bool = True) -> np.ndarray:
    n = x.shape[0]
    sq = (x * x).sum(1)
    out = np.empty((n, j), np.int32)
    for lo in range(0, n, 2048):
        hi = min(lo + 2048, n)
        d2 = sq[None, :] - 2.0 * (x[lo:hi] @ x.T)
        if exclude_self:
            d2[np.arange(hi - lo), np.arange(lo, hi)] = np.inf
        part = np.argpartition(d2, j, axis=1)[:, :j]
        dd = np.take_along_axis(d2, part, 1)
        order = np.argsort(dd, axis=1, kind="stable")
        out[lo:hi] = np.take_along_axis(part, order, 1)
    return out


def nearest_in(src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    sq = (dst * dst).sum(1)
    out = np.empty(src.shape[0], np.int32)
    for lo in range(0, src.shape[0], 4096):
        hi = min(lo + 4096, src.shape[0])
        out[lo:hi] = np.argmin(sq[None, :] - 2.0 * (src[lo:hi] @ dst.T), axis=1)
    return out


def make_contexts(base: np.ndarray, n_shards: int, j: int, ghost_every: int = 50, j_g: int = 16,
                  seed: int = 0) -> list:
    n = base.shape[0]
    perm = np.random.default_rng(seed).permutation(n)
    rows = [np.sort(perm[s::n_shards]) for s in range(n_shards)]
    vecs = [np.ascontiguousarray(base[r]) for r in rows]
    ctxs = []
    for s in range(n_shards):
        v = vecs[s]
        adj = knn_graph(v, j)
        inter = nearest_in(v, vecs[(s + 1) % n_shards]) if n_shards > 1 else None
        gids = np.arange(0, v.shape[0], ghost_every, dtype=np.int32)
        ghost = None
        if gids.size > j_g:
            gadj = knn_graph(np.ascontiguousarray(v[gids]), j_g)
            ghost = GhostContext(vectors=np.ascontiguousarray(v[gids]), adj=gadj, parent_ids=gids)
        ctxs.append(ShardContext(vectors=v, adj=adj, global_ids=rows[s].astype(np.int32),
                                 direction=direction_table(v, adj), inter_map=inter, ghost=ghost))
    return ctxs
