"""Device-resident search driver (shards built from torch tensors, outputs kept
in HBM).  Same stage schedule as pipeline.run_* (pipeline.py:270-350), issued
as asynchronous pw_search_stage launches on one CUDA stream; used by bench.py
for the kernel-only timing and by ring.py for one-shard-per-GPU runs.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _abi

STAT_I32 = ("iterations", "ghost_iterations", "retained", "converged")
STAT_I64 = ("distance_computations", "total_visits", "inserted", "dgs_skipped",
            "nodes_expanded", "ghost_nodes_expanded")


def _ptr(t):
    return None if t is None else t.data_ptr()


class TensorShard:
    """A pw_shard created from device tensors (copied device-to-device)."""

    def __init__(self, vectors: torch.Tensor, adj: torch.Tensor, global_ids: torch.Tensor,
                 direction: torch.Tensor | None = None, inter_map: torch.Tensor | None = None,
                 ghost_ids: torch.Tensor | None = None, ghost_adj: torch.Tensor | None = None):
        lib = _abi.load()
        torch.cuda.set_device(vectors.device)
        self.device = vectors.device
        # uint8 rows stay uint8 on the device (the reference upcasts them,
        # data.py:36; float(b) is exact); anything else is float32
        vec = vectors.contiguous() if vectors.dtype == torch.uint8 else vectors.contiguous().float()
        self.dtype = "u8" if vec.dtype == torch.uint8 else "f32"
        adj = adj.contiguous().to(torch.int32)
        gid = global_ids.contiguous().to(torch.int32)
        dr = None if direction is None else direction.contiguous().to(torch.int32)
        it = None if inter_map is None else inter_map.contiguous().to(torch.int32)
        gi = None if ghost_ids is None else ghost_ids.contiguous().to(torch.int32)
        ga = None if ghost_adj is None else ghost_adj.contiguous().to(torch.int32)
        torch.cuda.synchronize(self.device)
        desc = _abi.ShardDesc(vec.shape[0], vec.shape[1], adj.shape[1], 1 if self.dtype == "u8" else 0,
                              _ptr(vec), _ptr(adj),
                              _ptr(gid), _ptr(dr), _ptr(it), 0 if gi is None else gi.shape[0],
                              0 if ga is None else ga.shape[1], _ptr(gi), _ptr(ga), 1)
        h = C.c_void_p()
        _abi.check(lib.pw_shard_create(C.byref(desc), C.byref(h)))
        self.handle = h
        self.n, self.d = vec.shape
        self.j = adj.shape[1]
        self.W = (self.d + 31) // 32
        self.ghost_n = 0 if gi is None else gi.shape[0]
        self.ghost_j = 0 if ga is None else ga.shape[1]
        self.has_inter = it is not None
        self.nbytes = int(lib.pw_shard_bytes(h))
        self._finalizer = weakref.finalize(self, lib.pw_shard_destroy, h)


def reduce_flag() -> torch.Tensor:
    """K2's error flag in page-locked host memory: K2 writes it through the
    unified address space (only when it fires), so checking it after the
    results were read back costs no extra device round trip."""
    return torch.zeros(1, dtype=torch.int32, pin_memory=True)


def check_reduce_flag(err: torch.Tensor, device=None) -> None:
    """Raise like pipeline.py:194 if a device-side K2 saw a query without any
    valid candidate; clears the flag.  Synchronises the device first."""
    torch.cuda.synchronize(device)
    if int(err[0]):
        err.zero_()
        raise ValueError("cannot reduce empty candidate lists")


def check_shard(shard: TensorShard) -> None:
    """Raise if the shard's device error flag is set (synchronises)."""
    _abi.check(_abi.load().pw_shard_check(shard.handle))


class DeviceRun:
    """Preallocated device outputs for Q queries over n_cols shard columns."""

    def __init__(self, q: int, n_cols: int, k: int, device):
        self.q, self.n_cols, self.k = q, n_cols, k
        dev = torch.device(device)
        self.shard_ids = torch.empty((q, n_cols, k), dtype=torch.int32, device=dev)
        self.shard_dists = torch.empty((q, n_cols, k), dtype=torch.float32, device=dev)
        self.final_ids = torch.empty((q, k), dtype=torch.int32, device=dev)
        self.final_dists = torch.empty((q, k), dtype=torch.float32, device=dev)
        self.s32 = torch.empty((n_cols, 4, q), dtype=torch.int32, device=dev)
        self.s64 = torch.empty((n_cols, 6, q), dtype=torch.int64, device=dev)
        # forwarded entries, up to 8 per query (tuning "forward_count", opt-in)
        self.entries = [torch.zeros(q * 8, dtype=torch.int32, device=dev) for _ in range(2)]
        self.err = reduce_flag()

    def reset(self, stream=None):
        """Padding (-1 / +inf) and zeroed StageStats, one launch on `stream`."""
        st = (stream or torch.cuda.current_stream(self.shard_ids.device)).cuda_stream
        _abi.check(_abi.load().pw_init_outputs(self.shard_ids.data_ptr(), self.shard_dists.data_ptr(),
                                               self.shard_ids.numel(), self.s32.data_ptr(), self.s32.numel(),
                                               self.s64.data_ptr(), self.s64.numel(), C.c_void_p(st)))

    def check(self) -> None:
        """Read and clear the K2 flag (synchronises): the device-resident
        reduce passes a device flag instead of synchronising, so the check
        happens where results are read back (pipeline.py:194)."""
        check_reduce_flag(self.err, self.final_ids.device)

    def stats(self) -> list[dict]:
        self.check()
        s32 = self.s32.cpu().numpy()
        s64 = self.s64.cpu().numpy()
        out = []
        for s in range(self.n_cols):
            st = {name: s32[s, i] for i, name in enumerate(STAT_I32)}
            st.update({name: s64[s, i] for i, name in enumerate(STAT_I64)})
            out.append(st)
        return out


def search_stage(shard: TensorShard, params, queries: torch.Tensor, q0: int, n: int, stage: int,
                 run: DeviceRun, col: int, stat_row: int, entries_in=None, forward_out=None,
                 tuning=None, stream=None) -> None:
    """One pw_search_stage launch (asynchronous on `stream`)."""
    lib = _abi.load()
    p = _abi.params_struct(params)
    t = _abi.tuning_struct(tuning)
    st = (stream or torch.cuda.current_stream(queries.device)).cuda_stream
    s32 = run.s32[stat_row]
    s64 = run.s64[stat_row]
    _abi.check(lib.pw_search_stage(shard.handle, C.byref(p), C.byref(t), queries.data_ptr(), q0, n,
                                   stage, _ptr(entries_in), _ptr(forward_out),
                                   run.shard_ids.data_ptr(), run.shard_dists.data_ptr(), run.n_cols,
                                   col, s32.data_ptr(), s64.data_ptr(), run.q, st))


def reduce(run: DeviceRun, stream=None) -> None:
    lib = _abi.load()
    st = (stream or torch.cuda.current_stream(run.final_ids.device)).cuda_stream
    _abi.check(lib.pw_reduce_topk(run.shard_ids.data_ptr(), run.shard_dists.data_ptr(), run.q,
                                  run.n_cols * run.k, run.k, run.final_ids.data_ptr(),
                                  run.final_dists.data_ptr(), run.err.data_ptr(), st))


def chunk_bounds(q: int, n: int) -> list[int]:
    """np.array_split(arange(q), n) boundaries (pipeline.py:327)."""
    lo = [0]
    for c in range(n):
        lo.append(lo[-1] + q // n + (1 if c < q % n else 0))
    return lo


def run_local(shards: list[TensorShard], params, queries: torch.Tensor, mode: str, run: DeviceRun,
              tuning=None, stream=None, timer: list | None = None, reduce_after=None) -> None:
    """All shards on this device: baseline (shard s = stage s, all queries) or
    pipelined (chunk c stage s on shard (c+s)%N, entry forwarded in HBM).
    If `timer` is a list, (start, end) CUDA events bracket every search launch.
    `params` may be a list of N SearchParams, one per stage (per-stage
    budgets, SPEC.md "a per-stage budget vector is configurable"; an opt-in
    extension -- the reference's run_pipelined uses one parameter set).
    `reduce_after`: a CUDA event the final reduce waits for (a reader of the
    previous batch's final lists on another stream)."""
    n = len(shards)
    per_stage = list(params) if isinstance(params, (list, tuple)) else [params] * n
    if len(per_stage) != n or len({p.k for p in per_stage}) != 1:
        raise ValueError("per-stage params: one SearchParams per stage, all with the same k")
    q = queries.shape[0]
    stream = stream or torch.cuda.current_stream(queries.device)

    def launch(*a, **kw):
        if timer is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        search_stage(*a, tuning=tuning, stream=stream, **kw)
        if timer is not None:
            e1.record(stream)
            timer.append((e0, e1))

    run.reset(stream)
    if mode == "baseline":
        for s in range(n):
            launch(shards[s], per_stage[s], queries, 0, q, s, run, s, s)
    else:
        lo = chunk_bounds(q, n)
        ein, eout = run.entries
        for stage in range(n):
            for c in range(n):
                shard = (c + stage) % n
                launch(shards[shard], per_stage[stage], queries, lo[c], lo[c + 1] - lo[c], stage, run, shard,
                       stage, entries_in=ein if stage > 0 else None,
                       forward_out=eout if stage < n - 1 else None)
            ein, eout = eout, ein
    if reduce_after is not None:
        stream.wait_event(reduce_after)
    reduce(run, stream)


class DevArray:
    """A pw_dev_alloc'd buffer (its own cudaMalloc, so a CUDA IPC handle maps
    exactly it) or an IPC mapping of another process's buffer, viewed as a
    torch tensor through __cuda_array_interface__ (no copy)."""

    _TYPESTR = {torch.int32: "<i4", torch.int64: "<i8", torch.float32: "<f4", torch.uint64: "<u8"}

    def __init__(self, shape, dtype, handle: bytes | None = None):
        lib = _abi.load()
        self.shape, self.dtype = tuple(shape), dtype
        nbytes = int(np.prod(self.shape)) * torch.empty((), dtype=dtype).element_size()
        ptr = C.c_void_p()
        if handle is None:
            _abi.check(lib.pw_dev_alloc(nbytes, C.byref(ptr)))
            self._finalizer = weakref.finalize(self, lib.pw_dev_free, ptr.value)
        else:
            buf = C.create_string_buffer(bytes(handle), 64)
            _abi.check(lib.pw_ipc_open(buf, C.byref(ptr)))
            self._finalizer = weakref.finalize(self, lib.pw_ipc_close, ptr.value)
        self.ptr = ptr.value
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": self._TYPESTR[dtype],
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        self.t = torch.as_tensor(self, device=torch.device("cuda", torch.cuda.current_device()))

    def ipc_handle(self) -> bytes:
        lib = _abi.load()
        buf = C.create_string_buffer(64)
        _abi.check(lib.pw_ipc_get(C.c_void_p(self.ptr), buf))
        return buf.raw


def search_dataflow(shard: TensorShard, params, queries: torch.Tensor, g: int, n: int, epoch: int,
                    inbox: int | None, next_inbox: int | None, shard_ids: int, shard_dists: int,
                    s32: int | None, s64: int | None, tuning=None, sm_limit: int = 0,
                    stream=None) -> None:
    """One pw_search_dataflow launch of shard g of an N-shard ring (device
    pointers; the inbox / outputs may be peer mappings)."""
    lib = _abi.load()
    p = _abi.params_struct(params)
    t = _abi.tuning_struct(tuning)
    st = (stream or torch.cuda.current_stream(queries.device)).cuda_stream
    _abi.check(lib.pw_search_dataflow(shard.handle, C.byref(p), C.byref(t), queries.data_ptr(),
                                      queries.shape[0], g, n, epoch & 0xFFFFFFFF, inbox, next_inbox,
                                      shard_ids, shard_dists, s32, s64, sm_limit, st))


class LocalDataflow:
    """The dataflow ring with all N shards on this GPU (logical shards): N
    persistent launches on N streams, each capped to SMs/N CTAs so that all
    are resident at once, entries handed over through device-memory inboxes.
    The same protocol as the one-GPU-per-shard ring (ring.DataflowRing),
    there over NVLink peer mappings."""

    def __init__(self, shards: list, q: int, k: int, device):
        self.shards = shards
        self.n = len(shards)
        dev = torch.device(device)
        # up to 8 entry words per query (tuning "forward_count", opt-in)
        self.inbox = [torch.zeros(q * 8, dtype=torch.int64, device=dev) for _ in range(self.n)]
        self.streams = [torch.cuda.Stream(dev) for _ in range(self.n)]
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.sm_limit = max(1, sms // self.n)
        self.epoch = 0

    def run(self, params, queries: torch.Tensor, run: DeviceRun, tuning=None, stream=None) -> None:
        stream = stream or torch.cuda.current_stream(queries.device)
        self.epoch += 1
        ready = torch.cuda.Event()
        ready.record(stream)
        done = []
        for g, sh in enumerate(self.shards):
            st = self.streams[g]
            st.wait_event(ready)
            search_dataflow(sh, params, queries, g, self.n, self.epoch, self.inbox[g].data_ptr(),
                            self.inbox[(g + 1) % self.n].data_ptr(), run.shard_ids.data_ptr(),
                            run.shard_dists.data_ptr(), run.s32.data_ptr(), run.s64.data_ptr(),
                            tuning=tuning, sm_limit=self.sm_limit, stream=st)
            ev = torch.cuda.Event()
            ev.record(st)
            done.append(ev)
        for ev in done:
            stream.wait_event(ev)
        reduce(run, stream)


def algorithmic_bytes(stats: list[dict], params, d: int, j: int, j_g: int, esize: int = 4,
                      seeded_stages: set | None = None) -> float:
    """Gather bytes the search path must read (per query summed):
    DC*d*s_e + (E + S)*j*4 + E_ghost*j_g*4 + P*j*W*4
    with P = pruned expansions = dgs_skipped / (j - n_keep) (each pruned parent
    reads its direction row, search.py:258) and S = 1 per neighbour-seeded
    search (adj[entry] read, pipeline.py:231).  Kernel-side re-reads (a
    parent's own vector for the DGS query bits, lossy-cache re-scores) are
    excluded, as §8(d) specifies."""
    W = (d + 31) // 32
    n_keep = max(1, int((1.0 - params.discard_ratio) * j + 0.5))
    total = 0.0
    for s, st in enumerate(stats):
        dc = float(st["distance_computations"].sum())
        e = float(st["nodes_expanded"].sum())
        eg = float(st["ghost_nodes_expanded"].sum())
        pruned = float(st["dgs_skipped"].sum()) / (j - n_keep) if j > n_keep else 0.0
        seeded = 0.0
        if params.seed_mode == "neighbors":
            seeded = float((st["ghost_iterations"] > 0).sum())
            if seeded_stages and s in seeded_stages:
                seeded = float(len(st["iterations"]))
        total += dc * d * esize + (e + seeded) * j * 4 + eg * j_g * 4 + pruned * j * W * 4
    return total
