"""GPU index builder for the benchmark inputs ("next" row).

The reference builds exact kNN graphs on the CPU (shardann/graphs.py:237-299),
O(n_local^2 d): 80-100 s at 100K points, days at 10M.  This module builds
the same *kinds* of structures on one B200 from torch tensors so the C2
workload (10M x 96) exists at all:

* ``partition``      balanced random partition (graphs.py:50-62 semantics:
                     permutation, shard s = sorted perm[s::N]) -- torch RNG,
                     not numpy's PCG64 stream, so shards differ from the
                     reference's for the same seed
* ``knn_graph``      approximate j-NN graph: IVF partition of the shard
                     (k-means centroids), each point scored exactly (fp32)
                     against the members of the `probe` clusters nearest to
                     its own centroid, then reverse-edge augmentation
                     (graphs.py:98-135: keep the best j of row U incoming)
* ``inter_shard``    nearest node of the next shard (graphs.py:138-154), same
                     IVF approximation
* ``ghost``          ceil(rho n) sampled nodes + their exact j_g-NN graph
                     (graphs.py:157-174)
* ``direction``      packed sign bits of every edge (graphs.py:177-186), exact
* ``exact_knn``      brute-force ground truth (oracle.py:48-69)

Graph quality affects recall, never parity: the search kernels are checked
against the oracle on whatever graph they are given.  GEMM screens use
torch/cuBLAS (a plain library GEMM on an offline path).
"""

from __future__ import annotations

import math

import numpy as np
import torch


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def gen_clustered(n: int, d: int, n_clusters: int, spread: float, seed: int,
                  device="cuda") -> torch.Tensor:
    """gen_synthetic's family (data.py:159-176): uniform centres in [0,1]^d,
    point i = centre[i % n_clusters] + spread * N(0, I); torch Philox RNG."""
    g = _gen(seed, device)
    centres = torch.rand((n_clusters, d), generator=g, device=device, dtype=torch.float32)
    out = torch.empty((n, d), device=device, dtype=torch.float32)
    step = 1 << 22
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        noise = torch.randn((hi - lo, d), generator=g, device=device, dtype=torch.float32)
        idx = torch.arange(lo, hi, device=device) % n_clusters
        out[lo:hi] = centres[idx] + noise * spread
    return out


def gen_latent(n: int, d: int, m: int, n_clusters: int, spread: float, noise: float, seed: int,
               device="cuda") -> torch.Tensor:
    """Low-intrinsic-dimension variant of the same clustered-Gaussian family:
    latent z = centre[i % n_clusters] + spread * N(0, I_m) in [0,1]^m, lifted to
    d dims by a fixed random linear map, plus isotropic noise.  Real descriptor
    sets (DEEP, SIFT) have intrinsic dimension far below d; this keeps graph
    navigation realistic at 10M points."""
    g = _gen(seed, device)
    centres = torch.rand((n_clusters, m), generator=g, device=device, dtype=torch.float32)
    lift = torch.randn((m, d), generator=g, device=device, dtype=torch.float32) / math.sqrt(m)
    out = torch.empty((n, d), device=device, dtype=torch.float32)
    step = 1 << 22
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        idx = torch.arange(lo, hi, device=device) % n_clusters
        z = centres[idx] + spread * torch.randn((hi - lo, m), generator=g, device=device)
        out[lo:hi] = z @ lift + noise * torch.randn((hi - lo, d), generator=g, device=device)
    return out


def partition(n: int, n_shards: int, seed: int, device="cuda") -> list[torch.Tensor]:
    perm = torch.randperm(n, generator=_gen(seed + 0x51, device), device=device)
    return [torch.sort(perm[s::n_shards]).values for s in range(n_shards)]


def _sqnorm(x: torch.Tensor) -> torch.Tensor:
    return (x * x).sum(1)


def _nearest_centroid(x: torch.Tensor, cent: torch.Tensor, chunk: int = 1 << 17) -> torch.Tensor:
    cn = _sqnorm(cent)
    out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    for lo in range(0, x.shape[0], chunk):
        hi = min(lo + chunk, x.shape[0])
        d2 = cn[None, :] - 2.0 * (x[lo:hi] @ cent.T)
        out[lo:hi] = torch.argmin(d2, dim=1)
    return out


def kmeans(x: torch.Tensor, n_lists: int, iters: int, seed: int) -> tuple[torch.Tensor, torch.Tensor]:
    n = x.shape[0]
    n_lists = min(n_lists, n)
    pick = torch.randperm(n, generator=_gen(seed + 0x1F, x.device), device=x.device)[:n_lists]
    cent = x[pick].clone()
    assign = _nearest_centroid(x, cent)
    for _ in range(iters):
        sums = _segment_sums(x, assign, n_lists)
        cnt = torch.bincount(assign, minlength=n_lists).to(torch.float64)
        keep = cnt > 0
        cent[keep] = (sums[keep] / cnt[keep, None]).to(cent.dtype)
        assign = _nearest_centroid(x, cent)
    return cent, assign


def _segment_sums(x: torch.Tensor, seg: torch.Tensor, n_seg: int) -> torch.Tensor:
    """Deterministic per-segment float64 sums: stable sort by segment, running
    float64 prefix sums, differences at segment ends (index_add_ uses atomics
    whose order, and therefore rounding, varies run to run)."""
    order = torch.sort(seg, stable=True).indices
    counts = torch.bincount(seg, minlength=n_seg)
    ends = torch.cumsum(counts, 0)                        # exclusive end of each segment
    at_end = torch.zeros((n_seg, x.shape[1]), dtype=torch.float64, device=x.device)
    carry = torch.zeros(x.shape[1], dtype=torch.float64, device=x.device)
    step = 1 << 21
    for lo in range(0, x.shape[0], step):
        hi = min(lo + step, x.shape[0])
        cs = torch.cumsum(x[order[lo:hi]].double(), 0) + carry
        carry = cs[-1]
        sel = (ends >= lo + 1) & (ends <= hi) & (counts > 0)
        at_end[sel] = cs[ends[sel] - 1 - lo]
    # prefix value at the end of the previous non-empty segment
    idx = torch.where(counts > 0, torch.arange(n_seg, device=x.device),
                      torch.full((n_seg,), -1, device=x.device, dtype=torch.int64))
    last = torch.cummax(idx, 0).values
    prefix = torch.where(last[:, None] >= 0, at_end[last.clamp(min=0)], torch.zeros_like(at_end))
    prev = torch.zeros_like(prefix)
    prev[1:] = prefix[:-1]
    return torch.where((counts > 0)[:, None], prefix - prev, torch.zeros_like(prefix))


class IVF:
    """Inverted lists of a base set: members sorted by list."""

    def __init__(self, base: torch.Tensor, n_lists: int, iters: int = 2, seed: int = 0):
        self.base = base
        self.cent, assign = kmeans(base, n_lists, iters, seed)
        self.order = torch.sort(assign, stable=True).indices
        counts = torch.bincount(assign, minlength=self.cent.shape[0])
        self.offsets = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=base.device)
        self.offsets[1:] = torch.cumsum(counts, 0)
        self.counts = counts

    def search(self, queries: torch.Tensor, k: int, probe: int, exclude: torch.Tensor | None = None,
               budget: int = 1 << 28) -> torch.Tensor:
        """Approximate top-k base ids per query (exact fp32 distances over the
        members of the `probe` lists nearest to the query's own list)."""
        dev = queries.device
        nq = queries.shape[0]
        L = self.cent.shape[0]
        probe = min(probe, L)
        qlist = _nearest_centroid(queries, self.cent)
        cn = _sqnorm(self.cent)
        lnbr = torch.empty((L, probe), dtype=torch.int64, device=dev)
        for lo in range(0, L, 4096):
            hi = min(L, lo + 4096)
            d2 = cn[None, :] - 2.0 * (self.cent[lo:hi] @ self.cent.T)
            lnbr[lo:hi] = torch.topk(d2, probe, dim=1, largest=False).indices
        qorder = torch.sort(qlist, stable=True).indices
        qcounts = torch.bincount(qlist, minlength=L)
        qoff = torch.zeros(L + 1, dtype=torch.int64, device=dev)
        qoff[1:] = torch.cumsum(qcounts, 0)
        ccount = self.counts[lnbr].sum(1)                      # candidates per list
        out = torch.full((nq, k), -1, dtype=torch.int64, device=dev)
        bn = _sqnorm(self.base)
        lists = torch.argsort(qcounts * ccount, descending=True)
        lists = lists[qcounts[lists] > 0]
        qc_h = qcounts[lists].cpu().numpy()
        cc_h = ccount[lists].cpu().numpy()
        i = 0
        nl = len(lists)
        while i < nl:
            M = int(qc_h[i])
            Nc = int(cc_h[i:i + 1].max())
            B = max(1, budget // max(1, M * Nc))
            B = min(B, nl - i)
            Nc = int(cc_h[i:i + B].max())
            sel = lists[i:i + B]
            # padded query ids (B, M)
            ar = torch.arange(M, device=dev)
            qs = qoff[sel][:, None] + ar[None, :]
            qmask = ar[None, :] < qcounts[sel][:, None]
            qids = qorder[torch.where(qmask, qs, qoff[sel][:, None])]
            # padded candidate ids (B, Nc): concatenation of the probe lists
            nb = lnbr[sel]                                      # (B, P)
            cnt = self.counts[nb]                               # (B, P)
            start = self.offsets[nb]
            cum = torch.cumsum(cnt, 1)
            pos = torch.arange(Nc, device=dev)
            seg = torch.searchsorted(cum, pos[None, :].expand(B, Nc).contiguous(), right=True)
            seg_c = seg.clamp(max=nb.shape[1] - 1)
            prev = torch.where(seg_c > 0, torch.gather(cum, 1, (seg_c - 1).clamp(min=0)),
                               torch.zeros_like(seg_c))
            within = pos[None, :] - prev
            cvalid = seg < nb.shape[1]
            cpos = torch.gather(start, 1, seg_c) + within
            cids = self.order[torch.where(cvalid, cpos, torch.zeros_like(cpos))]
            xq = queries[qids]                                  # (B, M, d)
            xb = self.base[cids]                                # (B, Nc, d)
            d2 = bn[cids][:, None, :] - 2.0 * torch.bmm(xq, xb.transpose(1, 2))
            d2 = d2 + _sqnorm(xq.reshape(-1, xq.shape[-1])).reshape(B, M)[:, :, None]
            d2.masked_fill_(~cvalid[:, None, :], float("inf"))
            if exclude is not None:
                d2.masked_fill_(exclude[qids][:, :, None] == cids[:, None, :], float("inf"))
            kk = min(k, Nc)
            top = torch.topk(d2, kk, dim=2, largest=False)
            ids = torch.gather(cids[:, None, :].expand(B, M, Nc), 2, top.indices)
            ids = torch.where(torch.isinf(top.values), torch.full_like(ids, -1), ids)
            flat_q = qids[qmask]
            out[flat_q, :kk] = ids[qmask]
            i += B
        return out


def reverse_augment(x: torch.Tensor, adj: torch.Tensor, chunk: int = 1 << 17) -> torch.Tensor:
    """graphs.py:110-134: best j of (row U incoming sources) by distance, with
    at most j incoming sources considered per node."""
    n, j = adj.shape
    dev = x.device
    src = torch.arange(n, device=dev, dtype=torch.int64).repeat_interleave(j)
    dst = adj.reshape(-1).to(torch.int64)
    valid = dst >= 0
    src, dst = src[valid], dst[valid]
    order = torch.argsort(dst, stable=True)
    dst_s, src_s = dst[order], src[order]
    starts = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    starts[1:] = torch.cumsum(torch.bincount(dst_s, minlength=n), 0)
    rank = torch.arange(dst_s.numel(), device=dev) - starts[dst_s]
    keep = rank < j
    rev = torch.full((n, j), -1, dtype=torch.int64, device=dev)
    rev[dst_s[keep], rank[keep]] = src_s[keep]
    del src, dst, order, dst_s, src_s, rank, keep
    out = torch.empty((n, j), dtype=torch.int32, device=dev)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        cand = torch.cat([adj[lo:hi].to(torch.int64), rev[lo:hi]], 1)   # (c, 2j)
        srt, _ = torch.sort(cand, 1)
        dup = torch.zeros_like(srt, dtype=torch.bool)
        dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
        bad = dup | (srt < 0) | (srt == torch.arange(lo, hi, device=dev)[:, None])
        safe = torch.where(bad, torch.zeros_like(srt), srt)
        diff = x[safe] - x[lo:hi][:, None, :]
        d2 = (diff * diff).sum(2)
        d2.masked_fill_(bad, float("inf"))
        top = torch.topk(d2, j, dim=1, largest=False)
        row = torch.gather(safe, 1, top.indices)
        # degree deficit: repeat the last valid neighbour (graphs.py:131-132)
        inf = torch.isinf(top.values)
        if inf.any():
            nvalid = (~inf).sum(1, keepdim=True).clamp(min=1)
            last = torch.gather(row, 1, nvalid - 1)
            row = torch.where(inf, last.expand_as(row), row)
        out[lo:hi] = row.to(torch.int32)
    return out


def knn_graph(x: torch.Tensor, j: int, probe: int = 8, n_lists: int | None = None,
              seed: int = 0, augment: bool = True, refine: int = 0) -> torch.Tensor:
    n = x.shape[0]
    if n <= 1 << 16:
        adj = exact_knn(x, x, j, exclude_self=True).to(torch.int32)
    else:
        n_lists = n_lists or max(64, int(n // 600))
        ivf = IVF(x, n_lists, iters=2, seed=seed)
        self_ids = torch.arange(n, device=x.device)
        adj = ivf.search(x, j, probe, exclude=self_ids).to(torch.int32)
        bad = adj < 0
        if bad.any():  # rows with too few candidates: fall back to repeating row[0]
            adj = torch.where(bad, adj[:, :1].expand_as(adj), adj)
        if refine:
            adj = refine_knn(x, adj, refine)
    return reverse_augment(x, adj) if augment else adj


def refine_knn(x: torch.Tensor, adj: torch.Tensor, iters: int = 1, chunk: int = 8192) -> torch.Tensor:
    """Neighbour-of-neighbour refinement of an approximate j-NN graph (one
    NN-descent style pass per iteration): each row keeps the j nearest of
    its neighbours and their neighbours.  Moves the IVF graph toward the
    reference's exact kNN graph (graphs.py:104-134)."""
    n, j = adj.shape
    dev = x.device
    for _ in range(iters):
        new = torch.empty_like(adj)
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            a = adj[lo:hi].long()
            cand = torch.cat([a, adj[a.reshape(-1)].long().reshape(hi - lo, j * j)], 1)
            cs = torch.sort(cand, 1).values
            drop = torch.zeros_like(cs, dtype=torch.bool)
            drop[:, 1:] = cs[:, 1:] == cs[:, :-1]
            drop |= cs == torch.arange(lo, hi, device=dev)[:, None]
            d2 = ((x[cs] - x[lo:hi, None, :]) ** 2).sum(-1)
            d2.masked_fill_(drop, float("inf"))
            top = torch.topk(d2, j, dim=1, largest=False).indices
            new[lo:hi] = torch.gather(cs, 1, top).to(adj.dtype)
        adj = new
    return adj


def exact_knn(base: torch.Tensor, queries: torch.Tensor, k: int, exclude_self: bool = False,
              qchunk: int = 4096, bchunk: int = 1 << 21) -> torch.Tensor:
    """Brute-force top-k ids (fp32), ties broken arbitrarily."""
    dev = base.device
    nq = queries.shape[0]
    bn = _sqnorm(base)
    out = torch.empty((nq, k), dtype=torch.int64, device=dev)
    for qlo in range(0, nq, qchunk):
        qhi = min(nq, qlo + qchunk)
        best_v = None
        best_i = None
        for blo in range(0, base.shape[0], bchunk):
            bhi = min(base.shape[0], blo + bchunk)
            d2 = bn[None, blo:bhi] - 2.0 * (queries[qlo:qhi] @ base[blo:bhi].T)
            if exclude_self:
                r = torch.arange(qlo, qhi, device=dev)
                m = (r >= blo) & (r < bhi)
                d2[m.nonzero().squeeze(1), (r[m] - blo)] = float("inf")
            kk = min(k, bhi - blo)
            t = torch.topk(d2, kk, dim=1, largest=False)
            v, i = t.values, t.indices + blo
            if best_v is None:
                best_v, best_i = v, i
            else:
                cv = torch.cat([best_v, v], 1)
                ci = torch.cat([best_i, i], 1)
                t2 = torch.topk(cv, min(k, cv.shape[1]), dim=1, largest=False)
                best_v, best_i = t2.values, torch.gather(ci, 1, t2.indices)
        out[qlo:qhi, : best_i.shape[1]] = best_i
    return out


def exact_knn_rescored(base: torch.Tensor, queries: torch.Tensor, k: int, pad: int = 8) -> torch.Tensor:
    """Ground truth: GEMM screen for k+pad candidates, exact fp32 rescore of
    (x-q)^2, rank by (distance, id) (oracle.py:37-69)."""
    cand = exact_knn(base, queries, k + pad)
    out = torch.empty((queries.shape[0], k), dtype=torch.int64, device=base.device)
    for lo in range(0, queries.shape[0], 4096):
        hi = min(lo + 4096, queries.shape[0])
        c = cand[lo:hi]
        diff = base[c] - queries[lo:hi][:, None, :]
        d2 = (diff * diff).sum(2).double()
        key = d2 * (1 << 0) + c.double() * 0  # distance first
        order = torch.argsort(c, 1)
        c2 = torch.gather(c, 1, order)
        d2s = torch.gather(d2, 1, order)
        o2 = torch.sort(d2s, dim=1, stable=True).indices      # stable: ties keep id order
        out[lo:hi] = torch.gather(c2, 1, o2)[:, :k]
        del key
    return out


def exact_mips_rescored(base: torch.Tensor, queries: torch.Tensor, k: int, pad: int = 8,
                        qchunk: int = 1024, bchunk: int = 1 << 21) -> torch.Tensor:
    """Inner-product ground truth (BASELINE C5): fp32 GEMM screen for the
    k+pad largest q.x, float64 rescore, rank by (-q.x, id)."""
    dev = base.device
    nq = queries.shape[0]
    kk = k + pad
    out = torch.empty((nq, k), dtype=torch.int64, device=dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for qlo in range(0, nq, qchunk):
            qhi = min(nq, qlo + qchunk)
            best_v = best_i = None
            for blo in range(0, base.shape[0], bchunk):
                bhi = min(base.shape[0], blo + bchunk)
                s = queries[qlo:qhi] @ base[blo:bhi].T
                t = torch.topk(s, min(kk, bhi - blo), dim=1, largest=True)
                v, i = t.values, t.indices + blo
                if best_v is not None:
                    v = torch.cat([best_v, v], 1)
                    i = torch.cat([best_i, i], 1)
                    t2 = torch.topk(v, min(kk, v.shape[1]), dim=1, largest=True)
                    v, i = t2.values, torch.gather(i, 1, t2.indices)
                best_v, best_i = v, i
            c = best_i
            sc = (base[c].double() * queries[qlo:qhi, None, :].double()).sum(2)
            order = torch.argsort(c, 1)
            c2 = torch.gather(c, 1, order)
            s2 = torch.gather(-sc, 1, order)
            o2 = torch.sort(s2, dim=1, stable=True).indices
            out[qlo:qhi] = torch.gather(c2, 1, o2)[:, :k]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def direction_table(x: torch.Tensor, adj: torch.Tensor, chunk: int = 1 << 16) -> torch.Tensor:
    """graphs.py:177-186: bit t of word t//32 = x[nbr][t] >= x[node][t]."""
    n, j = adj.shape
    d = x.shape[1]
    W = (d + 31) // 32
    out = torch.empty((n, j, W), dtype=torch.int32, device=x.device)
    weights = (torch.ones(32, dtype=torch.int64, device=x.device) << torch.arange(32, device=x.device))
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        bits = x[adj[lo:hi].to(torch.int64)] >= x[lo:hi][:, None, :]          # (c, j, d)
        if W * 32 != d:
            bits = torch.cat([bits, torch.zeros(bits.shape[:-1] + (W * 32 - d,), dtype=torch.bool,
                                                device=x.device)], -1)
        words = (bits.view(hi - lo, j, W, 32).to(torch.int64) * weights).sum(-1)
        out[lo:hi] = (words - ((words >> 31) << 32)).to(torch.int32)          # uint32 bits in int32
    return out


def ghost(x: torch.Tensor, rho: float, j_g: int, seed: int) -> tuple[torch.Tensor, torch.Tensor] | None:
    """graphs.py:157-174: ceil(rho n) sorted distinct samples + exact j_g-NN graph."""
    n = x.shape[0]
    g = int(math.ceil(rho * n - 1e-9))
    if g <= j_g:
        return None
    ids = torch.sort(torch.randperm(n, generator=_gen(seed + 0x33, x.device), device=x.device)[:g]).values
    gx = x[ids].contiguous()
    if g <= 1 << 17:
        gadj = exact_knn(gx, gx, j_g, exclude_self=True).to(torch.int32)
    else:
        gadj = knn_graph(gx, j_g, seed=seed, augment=False)
    return ids.to(torch.int32), gadj.to(torch.int32)


def inter_shard(src: torch.Tensor, dst: torch.Tensor, probe: int = 8, seed: int = 0) -> torch.Tensor:
    """graphs.py:138-154: nearest node of the next shard for every node."""
    if dst.shape[0] <= 1 << 16:
        return exact_knn(dst, src, 1)[:, 0].to(torch.int32)
    ivf = IVF(dst, max(64, dst.shape[0] // 600), iters=2, seed=seed)
    return ivf.search(src, 1, probe)[:, 0].clamp(min=0).to(torch.int32)


def recall_at_k(found: np.ndarray, truth: np.ndarray, k: int) -> float:
    """oracle.py:72-84 mean recall@k (id-set intersection)."""
    hits = 0
    for f, t in zip(found, truth):
        hits += len(set(f[:k][f[:k] >= 0].tolist()) & set(t[:k].tolist()))
    return hits / (k * len(truth))
