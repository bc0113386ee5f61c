"""Multi-shard orchestration on the B200 (drop-in for shardann/pipeline.py).

* ``build_contexts``      pipeline.py:121-155 (+ device upload, cached on each context)
* ``run_ghost_stage``     pipeline.py:158-184 (ghost search in one warp of K1)
* ``reduce_topk``         pipeline.py:187-196 (K2 on the device)
* ``run_sharded_baseline`` pipeline.py:270-305 (every shard searches every query)
* ``run_pipelined``       pipeline.py:308-350 (ring: chunk c stage s on shard (c+s)%N)

All shards of one call live on the current CUDA device (logical shards); one
shard per GPU over NCCL is ``paper_2507_17094_b200.ring``.  ``threads`` is
accepted for signature compatibility and never changes results (the
reference's own contract, pipeline.py:12-16).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .search import (
    GhostContext,
    SearchCounters,
    SearchParams,
    ShardContext,
    _search_device,
    device_shard,
)


@dataclass(frozen=True)
class StageMessage:
    """pipeline.py:43-58: one 4-byte entry id per query of a chunk."""

    stage: int
    chunk: int
    entries: np.ndarray | None

    @property
    def payload_bytes(self) -> int:
        return 0 if self.entries is None else 4 * len(self.entries)


@dataclass
class StageStats:
    """pipeline.py:61-85."""

    iterations: np.ndarray
    ghost_iterations: np.ndarray
    distance_computations: np.ndarray
    total_visits: np.ndarray
    inserted: np.ndarray
    retained: np.ndarray
    dgs_skipped: np.ndarray
    converged: np.ndarray

    @classmethod
    def empty(cls, q: int) -> "StageStats":
        return cls(
            iterations=np.zeros(q, np.int32), ghost_iterations=np.zeros(q, np.int32),
            distance_computations=np.zeros(q, np.int64), total_visits=np.zeros(q, np.int64),
            inserted=np.zeros(q, np.int64), retained=np.zeros(q, np.int32),
            dgs_skipped=np.zeros(q, np.int64), converged=np.zeros(q, bool))


@dataclass
class PipelineResult:
    """pipeline.py:88-118."""

    mode: str
    k: int
    shard_ids: np.ndarray
    shard_dists: np.ndarray
    final_ids: np.ndarray
    final_dists: np.ndarray
    stages: list
    comm_stage_bytes: np.ndarray

    @property
    def n_queries(self) -> int:
        return self.shard_ids.shape[0]

    @property
    def comm_bytes_per_link(self) -> np.ndarray:
        return self.comm_stage_bytes.sum(axis=0)

    @property
    def comm_bytes_total(self) -> int:
        return int(self.comm_stage_bytes.sum())

    def neighbor_lists(self) -> list:
        out = []
        for qi in range(self.n_queries):
            valid = self.final_ids[qi] >= 0
            out.append(NeighborList(qi, self.final_ids[qi][valid], self.final_dists[qi][valid]))
        return out


@dataclass(frozen=True)
class NeighborList:
    """oracle.py:20-34 (the result type PipelineResult.neighbor_lists returns)."""

    query_id: int
    ids: np.ndarray
    dists: np.ndarray


def build_contexts(index, dataset) -> list[ShardContext]:
    """pipeline.py:121-155, then upload every shard to the current device."""
    if dataset.d != index.d:
        raise ValueError(f"dataset d={dataset.d} does not match index d={index.d}")
    if dataset.n != index.n_total:
        raise ValueError(f"dataset n={dataset.n} does not match index n={index.n_total}")
    order = np.argsort(dataset.ids, kind="stable")
    sorted_ids = dataset.ids[order]
    contexts = []
    for pack in index.shards:
        pos = np.searchsorted(sorted_ids, pack.global_ids)
        if pos.max(initial=-1) >= dataset.n or not np.array_equal(sorted_ids[pos], pack.global_ids):
            raise ValueError("index global ids not present in dataset")
        rows = order[pos]
        vectors = np.ascontiguousarray(dataset.data[rows])
        ghost = None
        if pack.ghost_ids is not None:
            ghost = GhostContext(vectors=np.ascontiguousarray(vectors[pack.ghost_ids]),
                                 adj=pack.ghost_adj, parent_ids=pack.ghost_ids)
        ctx = ShardContext(vectors=vectors, adj=pack.adj, global_ids=pack.global_ids,
                           direction=pack.direction, inter_map=pack.inter_map, ghost=ghost)
        device_shard(ctx)
        contexts.append(ctx)
    return contexts


def run_ghost_stage(query, ctx, params: SearchParams, *, rng, query_id: int = 0):
    """pipeline.py:158-184: ghost search -> (parent-local entry id, counters)."""
    if getattr(ctx, "ghost", None) is None:
        raise ValueError("ghost index absent for this shard")
    gparams = params.with_(k=1, max_iter=params.ghost_max_iter, selection="full",
                           discard_ratio=0.0, ghost_enabled=False, log_visits=False,
                           buffer_cap=None)
    query = np.asarray(query, dtype=np.float32)
    if query.shape != (ctx.vectors.shape[1],):
        raise ValueError(
            f"query dimension {query.shape} does not match shard d={ctx.vectors.shape[1]}")
    res = _search_device(device_shard(ctx), True, query, gparams, (), rng, query_id)
    return int(res.ids[0]), res.counters


def reduce_topk(ids: np.ndarray, dists: np.ndarray, k: int):
    """pipeline.py:187-196 on the device (K2)."""
    import torch

    lib = _abi.load()
    ids = np.ascontiguousarray(np.asarray(ids).ravel(), np.int32)
    dists = np.ascontiguousarray(np.asarray(dists).ravel(), np.float32)
    if ids.size == 0 or not (ids >= 0).any():
        raise ValueError("cannot reduce empty candidate lists")
    dev = torch.device("cuda", torch.cuda.current_device())
    ti = torch.from_numpy(ids).to(dev)
    td = torch.from_numpy(dists).to(dev)
    oi = torch.empty(k, dtype=torch.int32, device=dev)
    od = torch.empty(k, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _abi.check(lib.pw_reduce_topk(ti.data_ptr(), td.data_ptr(), 1, ids.size, k, oi.data_ptr(),
                                  od.data_ptr(), None, stream))
    oi, od = oi.cpu().numpy(), od.cpu().numpy()
    n = int((oi >= 0).sum())
    return oi[:n].astype(np.int32), od[:n].astype(np.float32)


STAT_I32 = ("iterations", "ghost_iterations", "retained", "converged")
STAT_I64 = ("distance_computations", "total_visits", "inserted", "dgs_skipped")


def _run(mode: str, queries, index, dataset, params: SearchParams, contexts, tuning=None):
    contexts = contexts if contexts is not None else build_contexts(index, dataset)
    n = len(contexts)
    if mode == "pipelined" and n > 1 and any(
            getattr(c, "inter_map", None) is None for c in contexts):
        raise ValueError("pipelined mode requires inter-shard tables for every shard")
    if (params.selection == "direction" and params.discard_ratio > 0.0
            and any(getattr(c, "direction", None) is None for c in contexts)):
        raise ValueError("direction table required for direction-guided selection")
    lib = _abi.load()
    devs = [device_shard(c) for c in contexts]
    qdata = np.ascontiguousarray(queries.data, np.float32)
    if qdata.shape[1] != devs[0].d:
        raise ValueError(f"query dimension {qdata.shape[1:]} does not match shard d={devs[0].d}")
    q = qdata.shape[0]
    k = int(params.k)
    handles = (C.c_void_p * n)(*[d.handle.value for d in devs])
    p = _abi.params_struct(params)
    t = _abi.tuning_struct(tuning)
    # one result block: pw_run copies the six arrays back in one transfer
    res = _abi.result_block(q, n, k)
    shard_ids, shard_dists = res["shard_ids"], res["shard_dists"]
    final_ids, final_dists = res["final_ids"], res["final_dists"]
    s32, s64 = res["s32"], res["s64"]
    comm = np.empty((n, n), np.int64)
    _abi.check(lib.pw_run(handles, n, C.byref(p), C.byref(t), qdata.ctypes.data, q,
                          _abi.MODE[mode], shard_ids.ctypes.data, shard_dists.ctypes.data,
                          final_ids.ctypes.data, final_dists.ctypes.data, s32.ctypes.data,
                          s64.ctypes.data, comm.ctypes.data))
    stages = []
    for s in range(n):
        st = StageStats(
            iterations=s32[s, 0].copy(), ghost_iterations=s32[s, 1].copy(),
            distance_computations=s64[s, 0].copy(), total_visits=s64[s, 1].copy(),
            inserted=s64[s, 2].copy(), retained=s32[s, 2].copy(),
            dgs_skipped=s64[s, 3].copy(), converged=s32[s, 3].astype(bool))
        stages.append(st)
    return PipelineResult(mode=mode, k=k, shard_ids=shard_ids, shard_dists=shard_dists,
                          final_ids=final_ids, final_dists=final_dists, stages=stages,
                          comm_stage_bytes=comm)


def run_sharded_baseline(queries, index, dataset, params: SearchParams, threads: int = 1,
                         contexts: list | None = None, *, tuning: dict | None = None
                         ) -> PipelineResult:
    """pipeline.py:270-305: independent random-seeded search in every shard."""
    return _run("baseline", queries, index, dataset, params, contexts, tuning)


def run_pipelined(queries, index, dataset, params: SearchParams, threads: int = 1,
                  contexts: list | None = None, *, tuning: dict | None = None) -> PipelineResult:
    """pipeline.py:308-350: ring-pipelined search, 4-byte entry forwarded per stage."""
    return _run("pipelined", queries, index, dataset, params, contexts, tuning)
