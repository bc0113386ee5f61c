"""Per-shard beam search on the B200 (drop-in for shardann/search.py).

Types mirror shardann/search.py:30-151 field for field; ``search`` mirrors
search.py:269-335 and runs as one warp of the sm_100a kernel K1
(csrc/beam_search.cuh) through ``pw_search_one``.  The numpy ``Generator``
passed as ``rng`` is consumed and advanced exactly as the reference would
advance it (device restatement of PCG64/SeedSequence/choice/permutation).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, replace

import numpy as np

from . import _abi

SELECTION_MODES = ("full", "direction", "random")
SEED_MODES = ("neighbors", "mixed")


@dataclass(frozen=True)
class SearchParams:
    """Knobs of one search (search.py:39-73), validated identically."""

    k: int = 10
    l: int = 64
    m: int = 64
    r: int = 8
    max_iter: int = 64
    seed: int = 0
    selection: str = "full"
    discard_ratio: float = 0.0
    cooldown_ratio: float = 0.3
    ghost_enabled: bool = False
    ghost_max_iter: int = 8
    seed_mode: str = "neighbors"
    buffer_cap: int | None = None
    log_visits: bool = False
    # extension beyond the reference (BASELINE C5): "ip" = inner product,
    # distance -(q . x) in the same pairwise order; "l2" is the reference's
    metric: str = "l2"

    def __post_init__(self):
        if not (1 <= self.k <= self.l and 1 <= self.r <= self.l):
            raise ValueError(f"need k <= l and r <= l, got k={self.k} l={self.l} r={self.r}")
        if self.m < 1 or self.max_iter < 1 or self.ghost_max_iter < 1:
            raise ValueError("m, max_iter and ghost_max_iter must be >= 1")
        if not 0.0 <= self.discard_ratio < 1.0:
            raise ValueError(f"discard_ratio must be in [0, 1), got {self.discard_ratio}")
        if not 0.0 <= self.cooldown_ratio <= 1.0:
            raise ValueError(f"cooldown_ratio must be in [0, 1], got {self.cooldown_ratio}")
        if self.selection not in SELECTION_MODES:
            raise ValueError(f"selection must be one of {SELECTION_MODES}")
        if self.seed_mode not in SEED_MODES:
            raise ValueError(f"seed_mode must be one of {SEED_MODES}")
        if self.metric not in ("l2", "ip"):
            raise ValueError("metric must be one of ('l2', 'ip')")

    def with_(self, **kw) -> "SearchParams":
        return replace(self, **kw)


@dataclass
class SearchCounters:
    """search.py:76-100."""

    iterations: int = 0
    distance_computations: int = 0
    total_visits: int = 0
    nodes_expanded: int = 0
    dgs_skipped: int = 0
    inserted_total: int = 0

    def merge(self, other: "SearchCounters") -> None:
        self.iterations += other.iterations
        self.distance_computations += other.distance_computations
        self.total_visits += other.total_visits
        self.nodes_expanded += other.nodes_expanded
        self.dgs_skipped += other.dgs_skipped
        self.inserted_total += other.inserted_total


@dataclass(frozen=True)
class SearchResult:
    """search.py:103-114."""

    query_id: int
    ids: np.ndarray
    dists: np.ndarray
    local_ids: np.ndarray
    converged: bool
    counters: SearchCounters
    retained: int
    visited_ids: np.ndarray | None = None


@dataclass(frozen=True)
class GhostContext:
    """search.py:117-127."""

    vectors: np.ndarray
    adj: np.ndarray
    parent_ids: np.ndarray


@dataclass(frozen=True)
class ShardContext:
    """search.py:130-151.  The device copy is attached lazily (device_shard)."""

    vectors: np.ndarray
    adj: np.ndarray
    global_ids: np.ndarray
    direction: np.ndarray | None = None
    inter_map: np.ndarray | None = None
    ghost: GhostContext | None = None

    @property
    def n_local(self) -> int:
        return self.vectors.shape[0]

    @property
    def degree(self) -> int:
        return self.adj.shape[1]

    def ghost_as_context(self) -> "ShardContext":
        g = self.ghost
        return ShardContext(vectors=g.vectors, adj=g.adj, global_ids=g.parent_ids)


def byte_rows(vec: np.ndarray) -> bool:
    """True when float32 rows hold only integers in [0, 255] (SIFT-style
    bvecs the reference upcast, data.py:36): the device can keep them as
    uint8 -- 4x fewer gather bytes -- and float(b) recovers every value
    exactly, so distances stay bit-identical."""
    if vec.dtype == np.uint8:
        return vec.shape[1] % 4 == 0
    if vec.shape[1] % 4 != 0 or vec.size == 0:
        return False
    return bool(np.all((vec >= 0) & (vec <= 255) & (vec == np.floor(vec))))


class DeviceShard:
    """Owner of one ``pw_shard`` (device copies of a ShardContext).

    storage: "auto" keeps byte-valued rows as uint8 on the device
    (``byte_rows``), "f32" always uploads float32, "u8" requires byte rows."""

    def __init__(self, ctx, device: int | None = None, storage: str = "auto"):
        import torch

        lib = _abi.load()
        if device is not None:
            torch.cuda.set_device(device)
        self.device = torch.cuda.current_device()
        raw = np.asarray(ctx.vectors)
        if storage not in ("auto", "f32", "u8"):
            raise ValueError("storage must be one of ('auto', 'f32', 'u8')")
        u8 = storage != "f32" and byte_rows(raw)
        if storage == "u8" and not u8:
            raise ValueError("storage='u8' needs integer rows in [0, 255] with d % 4 == 0")
        vec = np.ascontiguousarray(raw, np.float32)
        vdev = np.ascontiguousarray(raw, np.uint8) if u8 else vec
        self.dtype = "u8" if u8 else "f32"
        adj = np.ascontiguousarray(ctx.adj, np.int32)
        if adj.ndim != 2:
            adj = adj.reshape(vec.shape[0], -1)
        gid = np.ascontiguousarray(ctx.global_ids, np.int32)
        direction = getattr(ctx, "direction", None)
        direction = None if direction is None else np.ascontiguousarray(direction, np.uint32)
        inter = getattr(ctx, "inter_map", None)
        inter = None if inter is None else np.ascontiguousarray(inter, np.int32)
        ghost = getattr(ctx, "ghost", None)
        gids = gadj = None
        if ghost is not None:
            gids = np.ascontiguousarray(ghost.parent_ids, np.int32)
            gadj = np.ascontiguousarray(ghost.adj, np.int32)
        if vec.shape[0] == 0:
            raise ValueError("empty graph")
        desc = _abi.ShardDesc(
            vec.shape[0], vec.shape[1], adj.shape[1], 1 if u8 else 0, vdev.ctypes.data, adj.ctypes.data,
            gid.ctypes.data, None if direction is None else direction.ctypes.data,
            None if inter is None else inter.ctypes.data,
            0 if gids is None else gids.shape[0], 0 if gadj is None else gadj.shape[1],
            None if gids is None else gids.ctypes.data, None if gadj is None else gadj.ctypes.data, 0)
        h = C.c_void_p()
        _abi.check(lib.pw_shard_create(C.byref(desc), C.byref(h)))  # validates every id range
        if ghost is not None and not np.array_equal(np.asarray(ghost.vectors, np.float32), vec[gids]):
            lib.pw_shard_destroy(h)
            raise ValueError("ghost vectors must be the parent shard's rows at parent_ids")
        self.handle = h
        self.n = vec.shape[0]
        self.d = vec.shape[1]
        self.j = adj.shape[1]
        self.has_direction = direction is not None
        self.has_inter = inter is not None
        self.ghost_n = 0 if gids is None else gids.shape[0]
        self.ghost_j = 0 if gadj is None else gadj.shape[1]
        self.nbytes = int(lib.pw_shard_bytes(h))
        self._finalizer = weakref.finalize(self, lib.pw_shard_destroy, h)

    def close(self) -> None:
        self._finalizer()


def device_shard(ctx) -> DeviceShard:
    """The DeviceShard attached to ``ctx`` (uploaded on first use)."""
    dev = ctx.__dict__.get("_pw_device")
    if dev is None:
        dev = DeviceShard(ctx)
        object.__setattr__(ctx, "_pw_device", dev)
    return dev


def _rng_in(rng) -> _abi.Rng:
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("rng must be a numpy Generator over PCG64 (shardann.rng.stream)")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = 2**64 - 1
    return _abi.Rng(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))


def _rng_out(rng, r: _abi.Rng) -> None:
    rng.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (r.state_hi << 64) | r.state_lo, "inc": (r.inc_hi << 64) | r.inc_lo},
        "has_uint32": int(r.has_uint32), "uinteger": int(r.uinteger)}


def _search_device(dev: DeviceShard, use_ghost: bool, query, params: SearchParams, seeds, rng,
                   query_id: int) -> SearchResult:
    lib = _abi.load()
    q = np.ascontiguousarray(query, np.float32)
    s = np.ascontiguousarray(np.asarray([int(x) for x in seeds], np.int64).reshape(-1))
    p = _abi.params_struct(params)
    r = _rng_in(rng)
    k = int(params.k)
    ids = np.empty(k, np.int32)
    dists = np.empty(k, np.float32)
    loc = np.empty(k, np.int32)
    out = _abi.SearchOut()
    cap = 0
    log = None
    if params.log_visits:
        n = dev.ghost_n if use_ghost else dev.n
        j = dev.ghost_j if use_ghost else dev.j
        want = min(int(params.m), n)
        per = min(int(params.buffer_cap or max(params.m, params.r * j)), int(params.r) * j)
        cap = min(n, want + (int(params.max_iter) - 1) * per)  # visited-set bound
        log = np.empty(max(cap, 1), np.int32)
    _abi.check(lib.pw_search_one(dev.handle, int(use_ghost), C.byref(p), q.ctypes.data,
                                 s.ctypes.data if s.size else None, int(s.size), C.byref(r),
                                 ids.ctypes.data, dists.ctypes.data, loc.ctypes.data, C.byref(out),
                                 None if log is None else log.ctypes.data, cap))
    _rng_out(rng, r)
    n = out.n_out
    counters = SearchCounters(out.iterations, out.distance_computations, out.total_visits,
                              out.nodes_expanded, out.dgs_skipped, out.inserted_total)
    visited = None
    if params.log_visits and out.n_visited:
        visited = log[: out.n_visited].copy()
    return SearchResult(query_id=query_id, ids=ids[:n].copy(), dists=dists[:n].copy(),
                        local_ids=loc[:n].copy(), converged=bool(out.converged), counters=counters,
                        retained=int(out.retained), visited_ids=visited)


def search(query, ctx, params: SearchParams, seeds=(), *, rng: np.random.Generator,
           query_id: int = 0) -> SearchResult:
    """One beam search over a shard (search.py:269-335) on the GPU."""
    if ctx.vectors.shape[0] == 0:
        raise ValueError("empty graph")
    query = np.asarray(query, dtype=np.float32)
    if query.shape != (ctx.vectors.shape[1],):
        raise ValueError(
            f"query dimension {query.shape} does not match shard d={ctx.vectors.shape[1]}")
    if (params.selection == "direction" and params.discard_ratio > 0.0
            and getattr(ctx, "direction", None) is None):
        raise ValueError("direction table required for direction-guided selection")
    n = ctx.vectors.shape[0]
    for s in seeds:
        if not 0 <= int(s) < n:
            raise ValueError(f"seed {int(s)} outside shard of {n} nodes")
    return _search_device(device_shard(ctx), False, query, params, seeds, rng, query_id)
