"""Multi-process ring (one shard per rank) over gloo on the CPU.

The GPU path drives the same schedule (ring.run_ring_pipelined) with NCCL
send/recv and the CUDA stage kernel; here each rank's stage is the CPU
oracle and the links are gloo, so the schedule, the 4-byte entry hand-off,
the column all-gather and the reduction are checked against the reference's
own outputs (golden small.npz, 4 shards -> world size 4) without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import STAT_FIELDS, expected, load, SMALL_BASE
from paper_2507_17094_b200 import ring
from paper_2507_17094_b200.search import SearchParams


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, arm, out_path):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z, base, queries, index, ctxs = load("small")
        ctx = ctxs[rank]
        q = queries.shape[0]
        k = 10
        params = SearchParams(**SMALL_BASE, **arm)
        shard_ids = np.full((q, world, k), -1, np.int32)
        shard_dists = np.full((q, world, k), np.inf, np.float32)
        s32 = np.zeros((world, 4, q), np.int32)
        s64 = np.zeros((world, 4, q), np.int64)
        ein = np.zeros(q, np.int32)
        eout = np.zeros(q, np.int32)

        def stage_fn(stage, q0, n, has_entries):
            oracle.run_stage(ctx, queries, q0, n, params, stage, ein if has_entries else None,
                             eout if stage < world - 1 else None, shard_ids, shard_dists, rank,
                             s32[stage], s64[stage], threads=1)
            return eout[q0:q0 + n].copy()

        def send_recv(payload, next_q0, next_n):
            recv = torch.empty(next_n, dtype=torch.int32)
            reqs = [dist.isend(torch.from_numpy(payload), (rank + 1) % world),
                    dist.irecv(recv, (rank - 1) % world)]
            for r in reqs:
                r.wait()
            ein[next_q0:next_q0 + next_n] = recv.numpy()

        if mode == "pipelined":
            ring.run_ring_pipelined(stage_fn, q, rank, world, send_recv)
        else:
            stage_fn(rank, 0, q, False)
        # all-gather this rank's column, sum the per-stage counters
        col_i = torch.from_numpy(np.ascontiguousarray(shard_ids[:, rank, :]))
        col_d = torch.from_numpy(np.ascontiguousarray(shard_dists[:, rank, :]))
        gi = [torch.empty_like(col_i) for _ in range(world)]
        gd = [torch.empty_like(col_d) for _ in range(world)]
        dist.all_gather(gi, col_i)
        dist.all_gather(gd, col_d)
        t32 = torch.from_numpy(s32)
        t64 = torch.from_numpy(s64)
        dist.all_reduce(t32)
        dist.all_reduce(t64)
        if rank == 0:
            full_i = torch.stack(gi, 1).numpy()
            full_d = torch.stack(gd, 1).numpy()
            final_i = np.full((q, k), -1, np.int32)
            final_d = np.full((q, k), np.inf, np.float32)
            for qi in range(q):
                ids, ds = oracle.reduce_topk(full_i[qi], full_d[qi], k)
                final_i[qi, :len(ids)] = ids
                final_d[qi, :len(ids)] = ds
            np.savez(out_path, shard_ids=full_i, shard_dists=full_d, final_ids=final_i,
                     final_dists=final_d, s32=t32.numpy(), s64=t64.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["pipelined", "baseline"])
@pytest.mark.parametrize("arm_idx", [0, 6])
def test_ring_over_gloo_matches_reference(tmp_path, mode, arm_idx):
    from golden_util import ARMS_SMALL

    arm = ARMS_SMALL[arm_idx]
    out = tmp_path / "ring.npz"
    world = 4
    mp.spawn(_worker, args=(world, _free_port(), mode, arm, str(out)), nprocs=world, join=True)
    got = np.load(out)
    z = load("small")[0]
    want = expected(z, f"arm{arm_idx:02d}_{mode}_")
    for key in ("final_ids", "final_dists", "shard_ids", "shard_dists"):
        assert np.array_equal(got[key], want[key]), key
    stats = {"iterations": got["s32"][:, 0], "ghost_iterations": got["s32"][:, 1],
             "retained": got["s32"][:, 2], "converged": got["s32"][:, 3],
             "distance_computations": got["s64"][:, 0], "total_visits": got["s64"][:, 1],
             "inserted": got["s64"][:, 2], "dgs_skipped": got["s64"][:, 3]}
    for f in STAT_FIELDS:
        assert np.array_equal(stats[f].astype(np.int64), want[f].astype(np.int64)), f
    comm = ring.comm_stage_bytes(want["final_ids"].shape[0], world) if mode == "pipelined" \
        else np.zeros((world, world), np.int64)
    assert np.array_equal(comm, want["comm"])

def test_ring_schedule_covers_every_chunk_once():
    for world in (1, 2, 3, 4, 8):
        for stage in range(world):
            chunks = sorted(ring.ring_schedule(g, world, stage) for g in range(world))
            assert chunks == list(range(world))
        for g in range(world):
            assert sorted(ring.ring_schedule(g, world, s) for s in range(world)) == list(range(world))


def test_comm_accounting_formula():
    """pipeline.py:340-341 / reference test_pipeline.py:78-91."""
    q, n = 100, 4
    comm = ring.comm_stage_bytes(q, n)
    sizes = [len(c) for c in np.array_split(np.arange(q), n)]
    for link in range(n):
        expect = sum(4 * sizes[c] for stage in range(n - 1) for c in range(n) if (c + stage) % n == link)
        assert comm.sum(axis=0)[link] == expect


def test_dataflow_task_order_is_a_valid_schedule():
    """Every shard runs every query exactly once; stage s of query q on shard
    g is fed by stage s-1 of q on shard g-1, which precedes it there."""
    for world in (1, 2, 3, 4, 8):
        for q in (1, 7, 100):
            lists = [ring.dataflow_tasks(g, world, q) for g in range(world)]
            for g, tasks in enumerate(lists):
                assert sorted(qid for _, qid in tasks) == list(range(q))
                assert [s for s, _ in tasks] == sorted(s for s, _ in tasks)  # stage-major
                pos = {t: i for i, t in enumerate(lists[(g - 1) % world])}
                for s, qid in tasks:
                    if s > 0:
                        assert (s - 1, qid) in pos


def _df_worker(rank, world, port, arm, out_path):
    """The dataflow protocol over gloo: per-query entry messages (isend, like
    the device's fire-and-forget inbox stores), tasks in dataflow order, the
    CPU oracle as the per-task search."""
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z, base, queries, index, ctxs = load("small")
        ctx = ctxs[rank]
        q = queries.shape[0]
        k = 10
        params = SearchParams(**SMALL_BASE, **arm)
        shard_ids = np.full((q, world, k), -1, np.int32)
        shard_dists = np.full((q, world, k), np.inf, np.float32)
        s32 = np.zeros((world, 4, q), np.int32)
        s64 = np.zeros((world, 4, q), np.int64)
        ein = np.zeros(q, np.int32)
        eout = np.zeros(q, np.int32)
        pending = []
        for stage, qid in ring.dataflow_tasks(rank, world, q):
            if stage > 0:
                msg = torch.empty(2, dtype=torch.int64)
                dist.recv(msg, (rank - 1) % world)
                assert int(msg[0]) == qid  # arrives in this shard's task order
                ein[qid] = int(msg[1])
            oracle.run_stage(ctx, queries, qid, 1, params, stage, ein if stage > 0 else None,
                             eout if stage < world - 1 else None, shard_ids, shard_dists, rank,
                             s32[stage], s64[stage], threads=1)
            if stage < world - 1:
                t = torch.tensor([qid, int(eout[qid])], dtype=torch.int64)
                pending.append((dist.isend(t, (rank + 1) % world), t))
        for w, _ in pending:
            w.wait()
        col_i = torch.from_numpy(np.ascontiguousarray(shard_ids[:, rank, :]))
        col_d = torch.from_numpy(np.ascontiguousarray(shard_dists[:, rank, :]))
        gi = [torch.empty_like(col_i) for _ in range(world)]
        gd = [torch.empty_like(col_d) for _ in range(world)]
        dist.all_gather(gi, col_i)
        dist.all_gather(gd, col_d)
        t32 = torch.from_numpy(s32)
        t64 = torch.from_numpy(s64)
        dist.all_reduce(t32)
        dist.all_reduce(t64)
        if rank == 0:
            full_i = torch.stack(gi, 1).numpy()
            full_d = torch.stack(gd, 1).numpy()
            final_i = np.full((q, k), -1, np.int32)
            final_d = np.full((q, k), np.inf, np.float32)
            for qi in range(q):
                ids, ds = oracle.reduce_topk(full_i[qi], full_d[qi], k)
                final_i[qi, :len(ids)] = ids
                final_d[qi, :len(ids)] = ds
            np.savez(out_path, shard_ids=full_i, shard_dists=full_d, final_ids=final_i,
                     final_dists=final_d, s32=t32.numpy(), s64=t64.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("arm_idx", [0, 6])
def test_dataflow_protocol_over_gloo_matches_reference(tmp_path, arm_idx):
    from golden_util import ARMS_SMALL

    arm = ARMS_SMALL[arm_idx]
    out = tmp_path / "df.npz"
    world = 4
    mp.spawn(_df_worker, args=(world, _free_port(), arm, str(out)), nprocs=world, join=True)
    got = np.load(out)
    want = expected(load("small")[0], f"arm{arm_idx:02d}_pipelined_")
    for key in ("final_ids", "final_dists", "shard_ids", "shard_dists"):
        assert np.array_equal(got[key], want[key]), key
    stats = {"iterations": got["s32"][:, 0], "ghost_iterations": got["s32"][:, 1],
             "retained": got["s32"][:, 2], "converged": got["s32"][:, 3],
             "distance_computations": got["s64"][:, 0], "total_visits": got["s64"][:, 1],
             "inserted": got["s64"][:, 2], "dgs_skipped": got["s64"][:, 3]}
    for f in STAT_FIELDS:
        assert np.array_equal(stats[f].astype(np.int64), want[f].astype(np.int64)), f
