"""Exact GPU index build and exact kNN ground truth -- the reference's
offline ``build_index`` (shardann/graphs.py:50-299) and ``exact_knn_batch``
(oracle.py:37-69), on the device.

Same recipe as the reference, B200-sized:

* screen: fp32 GEMM distances ``|x|^2 - 2 q.x`` (cuBLAS, TF32 off), blocked,
  keeping the ``k + PAD`` best candidates per row (graphs.py:65-78 keeps
  ``k + 8``; the larger pad only makes the screen safer);
* rescore: every candidate pair through ``pw_l2_pairs``, the numpy-pairwise
  float32 distance bit-identical to ``data.py:70-79``;
* rank by (distance, id) (graphs.py:97-100 ``lexsort``), self excluded.

Whenever the screen's candidates contain the exact neighbours -- the
reference makes the same assumption (graphs.py:3-9) -- every array equals
the reference's bit for bit: adjacency, reverse augmentation
(graphs.py:103-134), inter-shard table (:138-154), ghost sample and graph
(:162-174, numpy streams drawn on the host exactly as the reference draws
them), direction table (:177-186).  ``tests/test_gpu_exact.py`` checks it
against the indexes the reference built for the golden fixtures.

The screen is O(n^2 d) GEMM work: minutes at a few million points, so the
10M+ bench configurations keep the approximate IVF builder (builder.py).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .graphs import Index, ShardPack
from .rng import TAG_GHOST_SAMPLE, TAG_PARTITION, stream

PAD = 16


def l2_pairs(a: torch.Tensor, b: torch.Tensor, ia: torch.Tensor, ib: torch.Tensor) -> torch.Tensor:
    """squared_l2(b[ib[t]], a[ia[t]]) for every t, bit-exact (pw_l2_pairs)."""
    lib = _abi.load()
    a = a.contiguous().float()
    b = b.contiguous().float()
    ia = ia.contiguous().to(torch.int64)
    ib = ib.contiguous().to(torch.int64)
    out = torch.empty(ia.shape[0], dtype=torch.float32, device=a.device)
    st = torch.cuda.current_stream(a.device).cuda_stream
    _abi.check(lib.pw_l2_pairs(a.data_ptr(), b.data_ptr(), a.shape[1], ia.data_ptr(), ib.data_ptr(),
                               ia.shape[0], out.data_ptr(), C.c_void_p(st)))
    return out


def _rank_keys(sq: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
    """(distance, id) as one int64 key: non-negative float bits are monotone."""
    return (sq.view(torch.int32).to(torch.int64) << 32) | ids.to(torch.int64)


def _screen(base: torch.Tensor, queries: torch.Tensor, kk: int, qchunk: int = 4096,
            bchunk: int = 1 << 20) -> torch.Tensor:
    """(q, kk) candidate ids by blocked GEMM screen (graphs.py:65-78)."""
    n = base.shape[0]
    kk = min(kk, n)
    bn = (base * base).sum(1)
    out = torch.empty((queries.shape[0], kk), dtype=torch.int64, device=base.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for qlo in range(0, queries.shape[0], qchunk):
            qhi = min(queries.shape[0], qlo + qchunk)
            best_v = best_i = None
            for blo in range(0, n, bchunk):
                bhi = min(n, blo + bchunk)
                d2 = bn[None, blo:bhi] - 2.0 * (queries[qlo:qhi] @ base[blo:bhi].T)
                t = torch.topk(d2, min(kk, bhi - blo), dim=1, largest=False)
                v, i = t.values, t.indices + blo
                if best_v is not None:
                    v = torch.cat([best_v, v], 1)
                    i = torch.cat([best_i, i], 1)
                    t2 = torch.topk(v, min(kk, v.shape[1]), dim=1, largest=False)
                    v, i = t2.values, torch.gather(i, 1, t2.indices)
                best_v, best_i = v, i
            out[qlo:qhi] = best_i
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


# K4 (csrc/knn_screen.cu) above this many screened pairs; below, the FP32
# GEMM screen is fast enough and needs no certification
TC_MIN_PAIRS = 1 << 30
TC_ERR = 2.0 ** -7.5   # |TF32 dot - exact| <= TC_ERR/2 * |q| |x| (generous; exact.py _certify)


def knn_screen_tc(base: torch.Tensor, queries: torch.Tensor, kc: int, self_off: int = -1):
    """K4 tensor-core screen: (nq, kc) int64 candidate ids (-1 = none) and
    their approximate |x|^2 - 2 q.x (TF32 operands, FP32 accumulation),
    unsorted; query row r skips base row r + self_off when self_off >= 0."""
    lib = _abi.load()
    base = base.contiguous().float()
    queries = queries.contiguous().float()
    nq, n, d = queries.shape[0], base.shape[0], base.shape[1]
    xn = (base * base).sum(1)
    ids = torch.empty((nq, kc), dtype=torch.int32, device=base.device)
    vals = torch.empty((nq, kc), dtype=torch.float32, device=base.device)
    st = torch.cuda.current_stream(base.device).cuda_stream
    _abi.check(lib.pw_knn_screen(queries.data_ptr(), nq, base.data_ptr(), n, d, xn.data_ptr(), int(self_off),
                                 kc, ids.data_ptr(), vals.data_ptr(), C.c_void_p(st)))
    return ids.to(torch.int64), vals, xn


def _certify(queries: torch.Tensor, base_norm_max: float, vals: torch.Tensor, kth_exact: torch.Tensor,
             full: torch.Tensor) -> torch.Tensor:
    """Rows whose exact top-k provably lies inside the screened candidates.

    Every non-candidate c has a screened value a_c >= tau (the list's worst),
    and |a_c - t_c| <= E with t_c = |x_c|^2 - 2 q.x_c in exact arithmetic.
    Columns with |x_c| > R = |q| + sqrt(D_k) + 1e-3 are farther than D_k (the
    k-th exact distance) by the triangle inequality; for the others E <=
    TC_ERR |q| R + 2^-15 (2 R^2 + 2 |q| R).  The f32 pairwise distance is
    within 2^-20 relative of the real one.  So if (|q|^2 + tau - E)(1 - 2^-20)
    > D_k, no non-candidate can enter the top k (strictly: no id tie-break
    can either)."""
    q64 = queries.double()
    qn2 = (q64 * q64).sum(1)
    qn = qn2.sqrt()
    tau = torch.where(torch.isfinite(vals), vals, torch.full_like(vals, -float("inf"))).max(1).values.double()
    dk = kth_exact.double()
    R = torch.clamp(qn + dk.clamp(min=0).sqrt() + 1e-3, max=float(base_norm_max) + 1e-3)
    E = TC_ERR * qn * R + 2.0 ** -15 * (2 * R * R + 2 * qn * R)
    ok = (qn2 + tau - E) * (1 - 2.0 ** -20) > dk * (1 + 2.0 ** -20)
    return ok | ~full  # a list that is not full holds every other row


def _rescore_rank(base, queries, cand, k, exclude_self):
    """Bit-exact rescore (pw_l2_pairs) + (distance, id) rank of candidates."""
    nq, c = cand.shape
    valid = cand >= 0
    cc = torch.where(valid, cand, torch.zeros_like(cand))
    qi = torch.arange(nq, device=base.device).repeat_interleave(c)
    sq = l2_pairs(queries, base, qi, cc.reshape(-1)).reshape(nq, c)
    bad = ~valid
    if exclude_self:
        bad |= cand == torch.arange(nq, device=base.device)[:, None]
    sq = torch.where(bad, torch.full_like(sq, float("inf")), sq)
    key = _rank_keys(sq, torch.where(valid, cand, torch.full_like(cand, (1 << 31) - 1)))
    order = torch.sort(key, dim=1).indices[:, :k]
    return torch.gather(cand, 1, order), torch.gather(sq, 1, order)


def exact_topk(base: torch.Tensor, queries: torch.Tensor, k: int, exclude_self: bool = False,
               pad: int = PAD, screen: str = "auto", stats: dict | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """k best rows of ``base`` per query by (exact squared L2, id): screen,
    bit-exact rescore, rank.  exclude_self: query i is base row i.

    screen: "fp32" (blocked FP32 GEMM + top-k), "tc" (K4 tensor-core screen,
    each row certified against the TF32 error bound; uncertified rows are
    redone by the FP32 screen), "auto" (tc for large problems)."""
    nq, n, d = queries.shape[0], base.shape[0], base.shape[1]
    kc = k + pad + (1 if exclude_self else 0)
    use_tc = screen == "tc" or (screen == "auto" and nq * n >= TC_MIN_PAIRS and kc <= 64 and d % 4 == 0)
    if not use_tc:
        cand = _screen(base, queries, kc)
        return _rescore_rank(base, queries, cand, k, exclude_self)
    kc = min(64, max(kc, k + 32))
    t0 = time.perf_counter()
    # the screen sees centred rows: distances are translation invariant and
    # the TF32 error bound scales with |q| |x|, so this tightens certification
    mu = base.double().mean(0).float()
    bc = base - mu
    qc = bc if (queries.data_ptr() == base.data_ptr() and queries.shape == base.shape) else queries - mu
    cand, vals, xn = knn_screen_tc(bc, qc, kc, 0 if exclude_self else -1)
    if stats is not None:
        torch.cuda.synchronize(base.device)
        t1 = time.perf_counter()
    ids, sq = _rescore_rank(base, queries, cand, k, exclude_self)
    full = (cand >= 0).all(1)
    ok = _certify(qc, float(xn.max().sqrt()), vals, sq[:, k - 1], full)
    del bc, qc
    redo = torch.nonzero(~ok).flatten()
    if stats is not None:
        torch.cuda.synchronize(base.device)
        stats.update(rows=nq, certified=int(ok.sum()), redone=int(redo.numel()), kc=kc,
                     screen_s=round(t1 - t0, 2), rescore_s=round(time.perf_counter() - t1, 2))
    if redo.numel():
        # FP32 screen for the uncertified rows (exclude_self: those rows'
        # own index in base is their query index)
        qs = queries[redo].contiguous()
        c2 = _screen(base, qs, k + pad + (1 if exclude_self else 0))
        i2, s2 = _rescore_rank(base, qs, c2, k, False) if not exclude_self else \
            _rescore_rank_self(base, qs, c2, k, redo)
        ids[redo] = i2
        sq[redo] = s2
        if stats is not None:
            torch.cuda.synchronize(base.device)
            stats["redo_s"] = round(time.perf_counter() - t0 - stats["screen_s"] - stats["rescore_s"], 2)
    return ids, sq


def _rescore_rank_self(base, qs, cand, k, rows):
    """_rescore_rank for a subset of query rows that are base rows `rows`."""
    nq, c = cand.shape
    qi = torch.arange(nq, device=base.device).repeat_interleave(c)
    sq = l2_pairs(qs, base, qi, cand.reshape(-1)).reshape(nq, c)
    sq = torch.where(cand == rows[:, None], torch.full_like(sq, float("inf")), sq)
    key = _rank_keys(sq, cand)
    order = torch.sort(key, dim=1).indices[:, :k]
    return torch.gather(cand, 1, order), torch.gather(sq, 1, order)


def _reverse_augment(x: torch.Tensor, adj: torch.Tensor) -> torch.Tensor:
    """graphs.py:103-134: each row becomes the j best of (row U incoming
    sources) \\ {self} by (distance, id); a row short of j repeats its last."""
    n, j = adj.shape
    dev = x.device
    src = torch.arange(n, device=dev).repeat_interleave(j)
    dst = adj.reshape(-1).to(torch.int64)
    a = torch.cat([src, dst])   # row
    b = torch.cat([dst, src])   # candidate (forward edge, or the source of an incoming one)
    keep = a != b
    key = torch.unique(a[keep] * n + b[keep])  # sorted, distinct pairs
    a, b = key // n, key % n
    sq = l2_pairs(x, x, a, b)   # squared_l2(x[b], x[a]), graphs.py:125
    order = torch.sort(_rank_keys(sq, b), stable=True).indices
    order = order[torch.sort(a[order], stable=True).indices]  # (row, distance, id)
    a, b = a[order], b[order]
    first = torch.searchsorted(a, torch.arange(n, device=dev))
    rank = torch.arange(a.shape[0], device=dev) - first[a]
    sel = rank < j
    out = torch.full((n, j), -1, dtype=torch.int64, device=dev)
    out[a[sel], rank[sel]] = b[sel]
    count = torch.clamp(torch.bincount(a, minlength=n), max=j)
    if bool((count < j).any()):  # degree deficit: repeat the last valid neighbour
        last = out[torch.arange(n, device=dev), (count - 1).clamp(min=0)]
        col = torch.arange(j, device=dev)[None, :]
        out = torch.where(col >= count[:, None], last[:, None], out)
    return out.to(torch.int32)


def build_knn_graph(x: torch.Tensor, j: int, stats: dict | None = None) -> torch.Tensor:
    """graphs.py:104-134 exact j-NN graph + reverse augmentation, (n, j) int32."""
    n = x.shape[0]
    if not 0 <= j < n:
        raise ValueError(f"need 0 <= j < n_local, got j={j}, n_local={n}")
    if j == 0:
        return torch.empty((n, 0), dtype=torch.int32, device=x.device)
    t0 = time.perf_counter()
    adj, _ = exact_topk(x, x, j, exclude_self=True, stats=stats)
    if stats is not None:
        torch.cuda.synchronize(x.device)
        t1 = time.perf_counter()
    out = _reverse_augment(x, adj)
    if stats is not None:
        torch.cuda.synchronize(x.device)
        stats.update(knn_s=round(t1 - t0, 2), augment_s=round(time.perf_counter() - t1, 2))
    return out


def build_inter_shard_table(src: torch.Tensor, dst: torch.Tensor) -> torch.Tensor:
    """graphs.py:138-154: exact nearest node of the next shard, (n,) int32."""
    if dst.shape[0] == 0:
        raise ValueError("empty target shard")
    if src.shape[1] != dst.shape[1]:
        raise ValueError("shards must share dimension")
    ids, _ = exact_topk(dst, src, 1)
    return ids[:, 0].to(torch.int32)


def ghost_count(n_local: int, rho: float) -> int:
    """graphs.py:157-159."""
    return int(math.ceil(rho * n_local - 1e-9))


def build_ghost_index(x: torch.Tensor, rho: float, j_g: int, seed: int,
                      shard: int = 0) -> tuple[np.ndarray, torch.Tensor]:
    """graphs.py:162-174: the sample is drawn on the host with the reference's
    own numpy stream; its exact graph is built on the device."""
    if not 0.0 < rho <= 1.0:
        raise ValueError(f"sampling ratio must be in (0, 1], got {rho}")
    n = x.shape[0]
    g = ghost_count(n, rho)
    if g <= j_g:
        raise ValueError(f"ghost sample of {g} too small for out-degree {j_g}")
    rng = stream(seed, TAG_GHOST_SAMPLE, shard)
    ghost_ids = np.sort(rng.choice(n, size=g, replace=False)).astype(np.int32)
    gid = torch.from_numpy(ghost_ids).to(x.device).to(torch.int64)
    return ghost_ids, build_knn_graph(x[gid].contiguous(), j_g)


def partition_rows(n: int, n_shards: int, seed: int) -> list[np.ndarray]:
    """graphs.py:50-62 (rows per shard; host numpy, the reference's stream)."""
    if not 1 <= n_shards <= n:
        raise ValueError(f"need 1 <= N <= n, got N={n_shards}, n={n}")
    perm = stream(seed, TAG_PARTITION).permutation(n)
    return [np.sort(perm[s::n_shards]) for s in range(n_shards)]


@dataclass
class BuildReport:
    """graphs.py:218-234 per-phase build times (seconds)."""

    base_graph: float = 0.0
    inter_shard: float = 0.0
    ghost: float = 0.0
    direction: float = 0.0
    per_shard: list = field(default_factory=list)

    @property
    def total(self) -> float:
        return self.base_graph + self.inter_shard + self.ghost + self.direction


def build_index(dataset, n_shards: int, j: int, seed: int, *, rho: float = 0.01,
                ghost_degree: int | None = None, with_ghost: bool = True,
                with_direction: bool = True, device=None) -> tuple[Index, BuildReport]:
    """graphs.py:237-299 on the GPU: same arguments, same Index."""
    from .builder import direction_table

    dev = torch.device(device or "cuda")
    data = np.ascontiguousarray(getattr(dataset, "data", dataset), np.float32)
    ids = getattr(dataset, "ids", None)
    ids = np.arange(data.shape[0], dtype=np.int32) if ids is None else np.asarray(ids, np.int32)
    rows = partition_rows(data.shape[0], n_shards, seed)
    j_g = min(j, 16) if ghost_degree is None else ghost_degree
    xs = torch.from_numpy(data if data.flags.writeable else data.copy()).to(dev)
    report = BuildReport()
    packs = []

    def timed(fn):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize(dev)
        return out, time.perf_counter() - t0

    for s in range(n_shards):
        r = torch.from_numpy(rows[s]).to(dev)
        x = xs[r].contiguous()
        times = {}
        adj, times["base_graph"] = timed(lambda: build_knn_graph(x, j))
        inter = None
        if n_shards > 1:
            nxt = xs[torch.from_numpy(rows[(s + 1) % n_shards]).to(dev)].contiguous()
            inter, times["inter_shard"] = timed(lambda: build_inter_shard_table(x, nxt))
            del nxt
        else:
            times["inter_shard"] = 0.0
        ghost_ids = ghost_adj = None
        if with_ghost and ghost_count(x.shape[0], rho) > j_g:
            (ghost_ids, ghost_adj), times["ghost"] = timed(lambda: build_ghost_index(x, rho, j_g, seed, shard=s))
        else:
            times["ghost"] = 0.0
        direction = None
        if with_direction:
            direction, times["direction"] = timed(lambda: direction_table(x, adj))
        else:
            times["direction"] = 0.0
        for key in ("base_graph", "inter_shard", "ghost", "direction"):
            setattr(report, key, getattr(report, key) + times[key])
        report.per_shard.append(times)
        packs.append(ShardPack(
            global_ids=ids[rows[s]].astype(np.int32),
            adj=adj.cpu().numpy(),
            inter_map=None if inter is None else inter.cpu().numpy(),
            ghost_ids=ghost_ids,
            ghost_adj=None if ghost_adj is None else ghost_adj.cpu().numpy(),
            direction=None if direction is None else direction.cpu().numpy().view(np.uint32)))
    return Index(d=data.shape[1], n_total=data.shape[0], shards=packs), report


def exact_knn_batch(base, queries, k: int, ids=None) -> tuple[np.ndarray, np.ndarray]:
    """oracle.py:52-69 exact kNN ground truth on the device: (ids (q, k) int32
    global ids, dists (q, k) float32 sqrt'd), ranked by (distance, id)."""
    data = np.ascontiguousarray(getattr(base, "data", base), np.float32)
    gids = getattr(base, "ids", None) if ids is None else ids
    q = np.ascontiguousarray(getattr(queries, "data", queries), np.float32)
    if q.ndim != 2 or q.shape[1] != data.shape[1]:
        raise ValueError(f"query dimension {q.shape} does not match dataset d={data.shape[1]}")
    if not 1 <= k <= data.shape[0]:
        raise ValueError(f"k must be in [1, {data.shape[0]}], got {k}")
    xb = torch.from_numpy(data if data.flags.writeable else data.copy()).cuda()
    xq = torch.from_numpy(q if q.flags.writeable else q.copy()).cuda()
    loc, sq = exact_topk(xb, xq, k)
    loc = loc.cpu().numpy()
    out_ids = loc.astype(np.int32) if gids is None else np.asarray(gids, np.int32)[loc]
    return out_ids, np.sqrt(sq.cpu().numpy())
