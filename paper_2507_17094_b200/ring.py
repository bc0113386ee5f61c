"""One shard per GPU: the ring of pipelining-based path extension
(shardann/pipeline.py:308-385) and the naive sharded baseline (:270-305)
across processes, one process per GPU over torch.distributed (NCCL on GPUs,
gloo in the CPU tests).

Pipelined schedule (pipeline.py:327-342): queries are split into N chunks;
at stage s rank g searches chunk (g - s) mod N on its shard g, then sends the
chunk's forward entries (inter_map_g[top1], one int32 per query -- the only
payload that crosses a link, pipeline.py:339-341) to rank g+1, which seeds
stage s+1 of the same chunk with them.  Every rank is busy at every stage.
After the last stage each rank holds the shard-g column of every query's
candidate list; an all-gather assembles the (Q, N, k) lists and K2 reduces
them (pipeline.py:249-267).  Baseline: every rank searches every query on
its shard (stage index = shard index), then the same all-gather + reduce.

The per-stage search is pluggable (``stage_fn``) so the CPU tests drive this
exact schedule with the oracle over gloo.
"""

from __future__ import annotations

import numpy as np


def _abi_forward_count(tuning) -> int:
    from ._abi import forward_count

    return forward_count(tuning)


def chunk_bounds(q: int, n: int) -> list[int]:
    """np.array_split(arange(q), n) boundaries (pipeline.py:327)."""
    lo = [0]
    for c in range(n):
        lo.append(lo[-1] + q // n + (1 if c < q % n else 0))
    return lo


def ring_schedule(rank: int, world: int, stage: int) -> int:
    """Chunk processed by `rank` at `stage`: shard (c + s) % N == rank."""
    return (rank - stage) % world


def comm_stage_bytes(q: int, world: int) -> np.ndarray:
    """pipeline.py:340-341 accounting: (N_stages, N) bytes sent by each shard."""
    lo = chunk_bounds(q, world)
    out = np.zeros((world, world), np.int64)
    for stage in range(world - 1):
        for c in range(world):
            out[stage, (c + stage) % world] = 4 * (lo[c + 1] - lo[c])
    return out


def run_ring_pipelined(stage_fn, q: int, rank: int, world: int, send_recv) -> None:
    """Drive this rank through the pipelined ring (pipeline.py:327-347).

    stage_fn(stage, q0, n, has_entries) searches chunk [q0, q0+n) on this
    rank's shard and returns its forward payload (inter_map[top1] per query);
    send_recv(payload, next_q0, next_n) sends the payload to rank+1 and
    receives, from rank-1, the entries of the chunk this rank searches next.
    """
    lo = chunk_bounds(q, world)
    for stage in range(world):
        c = ring_schedule(rank, world, stage)
        fwd = stage_fn(stage, lo[c], lo[c + 1] - lo[c], stage > 0)
        if stage < world - 1:
            cn = ring_schedule(rank, world, stage + 1)
            send_recv(fwd, lo[cn], lo[cn + 1] - lo[cn])


def dataflow_tasks(rank: int, world: int, q: int) -> list[tuple[int, int]]:
    """The (stage, query) task list of one shard in the dataflow ring, in the
    order the persistent kernel takes them (pw_search_dataflow: df_base /
    df_lo): stage-major, stage s covering chunk (rank - s) mod N in query
    order.  Stage-0 tasks need no input; a stage-s task's entry comes from
    the previous shard's stage s-1 task of the same query, which that shard
    takes earlier in its own stage-major order -- so waits never form a cycle."""
    lo = chunk_bounds(q, world)
    out = []
    for stage in range(world):
        c = ring_schedule(rank, world, stage)
        out += [(stage, qid) for qid in range(lo[c], lo[c + 1])]
    return out


def validate_inter(shard, n_next: int) -> None:
    """The forwarded entries (inter_map[top1], pipeline.py:339) index the next
    rank's shard: reject an inter_map with ids outside [0, n_next) up front
    (they would be gather indices on the next GPU)."""
    from . import _abi

    _abi.check(_abi.load().pw_shard_validate_inter(shard.handle, int(n_next)))


class RingSearch:
    """Device engine of one rank (one shard on this GPU)."""

    def __init__(self, shard, q: int, k: int, rank: int, world: int, device, tuning=None):
        import torch

        from . import device as dv

        self.shard, self.q, self.k, self.rank, self.world = shard, q, k, rank, world
        self.tuning = tuning
        self.dev = torch.device(device)
        self.run_buf = dv.DeviceRun(q, world, k, self.dev)
        self.stream = torch.cuda.current_stream(self.dev)
        self._lib = None
        self.gloo = False
        if world == 1:
            # submit()'s final-id copies go to the host on a side stream, so
            # batch b+1's K1 starts right after batch b's reduce; batch b+1's
            # reduce waits for that copy before overwriting the lists.  Made
            # here: the first stream from torch's pool and the page-locked
            # buffer cost milliseconds once.
            self._d2h = torch.cuda.Stream(self.dev)
            self._ev_reduced = torch.cuda.Event()
            self._ev_copied = torch.cuda.Event()
            self._ev_copied.record(self._d2h)
            self.host_ids = torch.empty((q, k), dtype=torch.int32, pin_memory=True)
        if world > 1:
            import torch.distributed as dist

            self.gloo = dist.get_backend() == "gloo"
            sizes = [None] * world
            dist.all_gather_object(sizes, int(shard.n))
            if shard.has_inter:
                validate_inter(shard, sizes[(rank + 1) % world])

    # ---------------------------------------------------------------- device path
    side_d2h = True  # final-id copies on a side stream (A/B: False = in stream order)

    def submit(self, queries, params, mode: str, timer: list | None = None) -> None:
        """One rank: enqueue a batch without host synchronisation; its final
        ids land in a page-locked host buffer (`host_ids` after `sync`).
        Consecutive batches reuse the device buffers in stream order, so the
        host prepares batch b+1 while batch b runs.  N > 1 pipelines through
        DataflowRing.submit."""
        import torch

        from . import device as dv

        if self.world != 1:
            raise ValueError("RingSearch.submit is the one-rank path; use DataflowRing for N > 1")
        R = self.run_buf
        if not self.side_d2h:
            dv.run_local([self.shard], params, queries, mode, R, tuning=self.tuning, stream=self.stream, timer=timer)
            if getattr(self, "host_ids", None) is None or tuple(self.host_ids.shape) != tuple(R.final_ids.shape):
                self.host_ids = torch.empty(tuple(R.final_ids.shape), dtype=torch.int32, pin_memory=True)
            with torch.cuda.stream(self.stream):
                self.host_ids.copy_(R.final_ids, non_blocking=True)
            return
        dv.run_local([self.shard], params, queries, mode, R, tuning=self.tuning, stream=self.stream, timer=timer,
                     reduce_after=self._ev_copied)
        if getattr(self, "host_ids", None) is None or tuple(self.host_ids.shape) != tuple(R.final_ids.shape):
            self.host_ids = torch.empty(tuple(R.final_ids.shape), dtype=torch.int32, pin_memory=True)
        self._ev_reduced.record(self.stream)
        self._d2h.wait_event(self._ev_reduced)
        with torch.cuda.stream(self._d2h):
            self.host_ids.copy_(R.final_ids, non_blocking=True)
        self._ev_copied.record(self._d2h)

    def sync(self) -> None:
        """Wait for the submitted batches; raise on a device-side error."""
        from . import device as dv

        self.stream.synchronize()
        if getattr(self, "_d2h", None) is not None:
            self._d2h.synchronize()
        self.run_buf.check()
        dv.check_shard(self.shard)

    def run(self, queries, params, mode: str, timer: list | None = None) -> np.ndarray | None:
        """Search all queries; returns final ids (Q, k) numpy on rank 0."""
        import torch
        import torch.distributed as dist

        from . import device as dv

        R = self.run_buf
        if self.world > 1 and _abi_forward_count(self.tuning) > 1:
            raise ValueError("forward_count > 1 needs the dataflow ring (PW_RING=dataflow)")
        if self.world == 1:
            dv.run_local([self.shard], params, queries, mode, R, tuning=self.tuning,
                         stream=self.stream, timer=timer, reduce_after=getattr(self, "_ev_copied", None))
            ids = R.final_ids.cpu().numpy()
            R.check()
            return ids

        R.reset()
        g, N = self.rank, self.world

        def launch(stage, q0, n, entries_in, forward_out):
            if timer is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
            dv.search_stage(self.shard, params, queries, q0, n, stage, R, g, stage,
                            entries_in=entries_in, forward_out=forward_out, tuning=self.tuning,
                            stream=self.stream)
            if timer is not None:
                e1.record(self.stream)
                timer.append((e0, e1))

        if mode == "baseline":
            launch(g, 0, self.q, None, None)
        else:
            ein, eout = R.entries

            def stage_fn(stage, q0, n, has_entries):
                launch(stage, q0, n, ein if has_entries else None, eout if stage < N - 1 else None)
                return eout[q0:q0 + n]

            def send_recv(payload, next_q0, next_n):
                # 4 B per query over NVLink (pipeline.py:339-341): NCCL P2P on the
                # compute stream's order, so stage s+1 starts when its entries land
                if self.gloo:  # host staging (gloo P2P is CPU-only)
                    buf = torch.empty(next_n, dtype=torch.int32)
                    reqs = [dist.isend(payload.cpu(), (g + 1) % N), dist.irecv(buf, (g - 1) % N)]
                    for w in reqs:
                        w.wait()
                    ein[next_q0:next_q0 + next_n].copy_(buf)
                    return
                ops = [dist.P2POp(dist.isend, payload, (g + 1) % N),
                       dist.P2POp(dist.irecv, ein[next_q0:next_q0 + next_n], (g - 1) % N)]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()

            run_ring_pipelined(stage_fn, self.q, g, N, send_recv)
        # all-gather this rank's column of the candidate lists, then reduce (K2)
        col_ids = R.shard_ids[:, g, :].contiguous()
        col_d = R.shard_dists[:, g, :].contiguous()
        if self.gloo:
            li = [torch.empty_like(col_ids.cpu()) for _ in range(N)]
            ld = [torch.empty_like(col_d.cpu()) for _ in range(N)]
            dist.all_gather(li, col_ids.cpu())
            dist.all_gather(ld, col_d.cpu())
            all_ids = torch.stack(li).to(self.dev)
            all_d = torch.stack(ld).to(self.dev)
        else:
            all_ids = torch.empty((N,) + tuple(col_ids.shape), dtype=col_ids.dtype, device=self.dev)
            all_d = torch.empty((N,) + tuple(col_d.shape), dtype=col_d.dtype, device=self.dev)
            dist.all_gather_into_tensor(all_ids, col_ids)
            dist.all_gather_into_tensor(all_d, col_d)
        R.shard_ids.copy_(all_ids.permute(1, 0, 2))
        R.shard_dists.copy_(all_d.permute(1, 0, 2))
        dv.reduce(R, self.stream)
        ids = R.final_ids.cpu().numpy() if self.rank == 0 else None
        R.check()
        return ids

    def last_stats(self) -> list[dict]:
        return self.run_buf.stats()

    # ---------------------------------------------------------------- host (e2e) path
    def run_host(self, queries_host: np.ndarray, params) -> dict:
        """End-to-end through the C ABI with host buffers (N=1: pw_run)."""
        import ctypes as C

        from . import _abi

        if self.world == 1:
            lib = _abi.load()
            q = queries_host.shape[0]
            k = int(params.k)
            # one page-locked result block, reused across calls: pw_run copies
            # it back in one transfer (pageable memory would go through a
            # driver bounce copy)
            key = (q, k)
            if getattr(self, "_host_out_key", None) != key:
                self._host_out = _abi.result_block(q, 1, k, pinned=True)
                self._host_out["comm"] = np.empty((1, 1), np.int64)
                self._host_out_key = key
            out = dict(self._host_out)
            handles = (C.c_void_p * 1)(self.shard.handle.value)
            cached = getattr(self, "_host_structs", None)
            if cached is None or cached[0] != params:
                # ctypes structs built once per parameter set, not per call
                cached = self._host_structs = (params, _abi.params_struct(params), _abi.tuning_struct(self.tuning))
            p, t = cached[1], cached[2]
            _abi.check(lib.pw_run(handles, 1, C.byref(p), C.byref(t), queries_host.ctypes.data, q,
                                  _abi.MODE["pipelined"], out["shard_ids"].ctypes.data,
                                  out["shard_dists"].ctypes.data, out["final_ids"].ctypes.data,
                                  out["final_dists"].ctypes.data, out["s32"].ctypes.data,
                                  out["s64"].ctypes.data, out["comm"].ctypes.data))
            out["bytes_out"] = sum(v.nbytes for key, v in out.items() if key not in ("comm", "_raw"))
            return out
        import torch

        qd = torch.from_numpy(queries_host).to(self.dev, non_blocking=False)
        ids = self.run(qd, params, "pipelined")
        out = {"final_ids": ids}
        if self.rank == 0:
            out["final_dists"] = self.run_buf.final_dists.cpu().numpy()
            out["bytes_out"] = out["final_ids"].nbytes + out["final_dists"].nbytes
        else:
            out["bytes_out"] = 0
        return out


class DataflowRing:
    """One shard per GPU, pipelined path extension WITHOUT stage barriers
    (pw_search_dataflow) and without host synchronisation between batches.

    Each rank runs one persistent K1 per batch over all its (stage, query)
    tasks; a finished stage-s search stores its entry (inter_map[top1],
    pipeline.py:339) straight into rank g+1's inbox -- a CUDA IPC peer
    mapping, so the 8-byte store travels over NVLink -- and writes its
    candidate-list column and counters straight into rank 0's result
    buffers.  Batches are double-buffered (``depth`` slots of inboxes and of
    rank 0's result buffers) and ordered on the device only:

    * every rank, after its K1 of batch e: ``pw_signal(landed[g][slot], e)``
      (a word in rank 0's memory);
    * rank 0: ``pw_wait(landed[*][slot] >= e)``, then K2 into the slot's
      final lists;
    * before a slot is reused by batch e + depth, rank 0 resets its buffers
      on its stream (after that slot's K2) and ``pw_signal(done[slot], e)``;
      every other rank ``pw_wait(done[slot] >= e)`` before its K1 of batch
      e + depth -- which also proves every rank consumed the slot's inboxes.

    ``submit`` only enqueues; ``result`` waits for one batch (rank 0).  So a
    stream of batches keeps every GPU busy: rank g starts batch e+1 while
    rank 0 still reduces batch e.  Baseline mode (naive sharding) uses the
    same slots with one pw_search_stage launch per rank.

    torch.distributed (NCCL or gloo) only carries the 64-byte IPC handles at
    construction.  Ranks may share a GPU (tests): pass sm_limit so every
    rank's persistent kernel stays resident."""

    def __init__(self, shard, q: int, k: int, rank: int, world: int, device, tuning=None,
                 sm_limit: int = 0, depth: int = 2):
        import torch
        import torch.distributed as dist

        from . import device as dv

        self.shard, self.q, self.k, self.rank, self.world = shard, q, k, rank, world
        self.tuning = tuning
        self.dev = torch.device(device)
        self.stream = torch.cuda.current_stream(self.dev)
        self.sm_limit = sm_limit
        self.depth = depth
        self.epoch = 0
        N = world
        self.inbox = dv.DevArray((depth, q * 8), torch.int64)  # <= 8 entry words per query
        res = flags = None
        if rank == 0:
            res = [[dv.DevArray((q, N, k), torch.int32), dv.DevArray((q, N, k), torch.float32),
                    dv.DevArray((N, 4, q), torch.int32), dv.DevArray((N, 6, q), torch.int64)]
                   for _ in range(depth)]
            flags = dv.DevArray((N + 1, depth), torch.int64)  # rows 0..N-1 landed[g], row N done
        handles = [None] * world
        mine = {"inbox": self.inbox.ipc_handle(), "n": int(shard.n),
                "res": [[a.ipc_handle() for a in slot] for slot in res] if res else None,
                "flags": flags.ipc_handle() if flags else None}
        dist.all_gather_object(handles, mine)
        nxt = (rank + 1) % world
        if world > 1:
            validate_inter(shard, handles[nxt]["n"])
        self.next_inbox = self.inbox if nxt == rank else dv.DevArray((depth, q * 8), torch.int64, handles[nxt]["inbox"])
        if rank == 0:
            self.res, self.flags = res, flags
        else:
            shapes = [((q, N, k), torch.int32), ((q, N, k), torch.float32), ((N, 4, q), torch.int32),
                      ((N, 6, q), torch.int64)]
            self.res = [[dv.DevArray(sh, dt, h) for (sh, dt), h in zip(shapes, slot)] for slot in handles[0]["res"]]
            self.flags = dv.DevArray((N + 1, depth), torch.int64, handles[0]["flags"])
        fp = self.flags.ptr
        row = depth * 8  # bytes per flags row

        def ptrs(lst):
            return torch.tensor(lst, dtype=torch.int64, device=self.dev)

        # device arrays of flag pointers for pw_wait, per slot
        self.landed_ptr = [fp + g * row + b * 8 for g in range(N) for b in range(depth)]
        self.landed_all = [ptrs([fp + g * row + b * 8 for g in range(N)]) for b in range(depth)]
        self.done_one = [ptrs([fp + N * row + b * 8]) for b in range(depth)]
        self.final_ids = [torch.empty((q, k), dtype=torch.int32, device=self.dev) for _ in range(depth)]
        self.final_dists = [torch.empty((q, k), dtype=torch.float32, device=self.dev) for _ in range(depth)]
        self.err = dv.reduce_flag()
        self.wait_err = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.ready = [torch.cuda.Event() for _ in range(depth)]
        self.last = 0
        if rank == 0:
            for b in range(depth):
                self._reset(b)
        torch.cuda.synchronize(self.dev)
        dist.barrier()  # buffers clean on rank 0 before any peer writes

    def _reset(self, b: int) -> None:
        ids, dists, s32, s64 = self.res[b]
        ids.t.fill_(-1)
        dists.t.fill_(float("inf"))
        s32.t.zero_()
        s64.t.zero_()

    def submit(self, queries, params, mode: str, timer: list | None = None) -> int:
        """Enqueue one batch (every rank passes the full (Q, d) device batch);
        returns its epoch.  No host synchronisation."""
        import ctypes as C

        import torch

        from . import _abi
        from . import device as dv

        lib = _abi.load()
        g, N, depth = self.rank, self.world, self.depth
        self.epoch += 1
        e = self.epoch
        b = e % depth
        ids, dists, s32, s64 = self.res[b]
        st = self.stream.cuda_stream
        if e > depth:  # the slot's previous batch (e - depth) must be reduced and its buffers reset
            if g == 0:
                self._reset(b)
                _abi.check(lib.pw_signal(self.flags.ptr + N * depth * 8 + b * 8, e - depth, st))
            else:
                _abi.check(lib.pw_wait(self.done_one[b].data_ptr(), 1, e - depth, self.wait_err.data_ptr(), st))
        e0 = e1 = None
        if timer is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        if mode == "baseline" or N == 1:
            # pipeline.py:288-297: every rank searches every query at stage g
            p = _abi.params_struct(params)
            t = _abi.tuning_struct(self.tuning)
            _abi.check(lib.pw_search_stage(self.shard.handle, C.byref(p), C.byref(t), queries.data_ptr(),
                                           0, self.q, g, None, None, ids.ptr, dists.ptr, N, g,
                                           s32.ptr + g * 4 * self.q * 4, s64.ptr + g * 6 * self.q * 8,
                                           self.q, st))
        else:
            dv.search_dataflow(self.shard, params, queries, g, N, e, self.inbox.ptr + b * self.q * 64,
                               self.next_inbox.ptr + b * self.q * 64, ids.ptr, dists.ptr, s32.ptr, s64.ptr,
                               tuning=self.tuning, sm_limit=self.sm_limit, stream=self.stream)
        if timer is not None:
            e1.record(self.stream)
            timer.append((e0, e1))
        _abi.check(lib.pw_signal(self.landed_ptr[g * depth + b], e, st))
        if g == 0:
            _abi.check(lib.pw_wait(self.landed_all[b].data_ptr(), N, e, self.wait_err.data_ptr(), st))
            _abi.check(lib.pw_reduce_topk(ids.ptr, dists.ptr, self.q, N * self.k, self.k,
                                          self.final_ids[b].data_ptr(), self.final_dists[b].data_ptr(),
                                          self.err.data_ptr(), st))
        self.ready[b].record(self.stream)
        self.last = e
        return e

    def _slot(self, e: int) -> int:
        if not (self.last - self.depth < e <= self.last):
            raise ValueError(f"batch {e} is no longer buffered (last {self.last}, depth {self.depth})")
        return e % self.depth

    def sync(self, e: int | None = None) -> None:
        """Wait for batch e (default: the last) on this rank and raise on any
        device-side error (a timed-out wait, a table overflow)."""
        from . import device as dv

        b = self._slot(self.last if e is None else e)
        self.ready[b].synchronize()
        if int(self.wait_err.item()):
            self.wait_err.zero_()
            raise RuntimeError("dataflow ring: a peer never signalled (pw_wait timed out)")
        dv.check_shard(self.shard)

    def result(self, e: int | None = None):
        """Final ids (Q, k) numpy of batch e (default: the last) on rank 0,
        None elsewhere."""
        from . import device as dv

        e = self.last if e is None else e
        self.sync(e)
        if self.rank != 0:
            return None
        ids = self.final_ids[self._slot(e)].cpu().numpy()
        dv.check_reduce_flag(self.err, self.dev)
        return ids

    def run(self, queries, params, mode: str, timer: list | None = None):
        """One batch, synchronously: final ids (Q, k) numpy on rank 0."""
        return self.result(self.submit(queries, params, mode, timer=timer))

    def last_final_dists(self):
        return self.final_dists[self.last % self.depth]

    def last_stats(self) -> list[dict]:
        from .device import STAT_I32, STAT_I64

        if self.rank != 0:
            return []
        self.sync()
        slot = self.res[self.last % self.depth]
        s32 = slot[2].t.cpu().numpy()
        s64 = slot[3].t.cpu().numpy()
        out = []
        for s in range(self.world):
            st = {name: s32[s, i] for i, name in enumerate(STAT_I32)}
            st.update({name: s64[s, i] for i, name in enumerate(STAT_I64)})
            out.append(st)
        return out

    def run_host(self, queries_host: np.ndarray, params) -> dict:
        """End to end: host queries in (H2D), final lists out on rank 0 (D2H)."""
        import torch

        qd = torch.from_numpy(queries_host).to(self.dev, non_blocking=False)
        ids = self.run(qd, params, "pipelined")
        out = {"final_ids": ids}
        if self.rank == 0:
            out["final_dists"] = self.last_final_dists().cpu().numpy()
            out["bytes_out"] = out["final_ids"].nbytes + out["final_dists"].nbytes
        else:
            out["bytes_out"] = 0
        return out
