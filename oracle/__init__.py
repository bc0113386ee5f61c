"""CPU oracle for the batched graph-ANNS search path -- TEST INFRASTRUCTURE.

This package is the parity checker, not the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It wraps ``liboracle.so``, a plain-C
restatement (``pw_oracle.c``) of the reference's search path:

* ``squared_l2``         shardann/data.py:70-79 (numpy pairwise float32 sum)
* ``derive_seed``/PCG64   shardann/rng.py:26-44 + numpy SeedSequence/PCG64
* ``choice``/``permutation`` numpy Generator.choice(replace=False)/permutation
* ``search``             shardann/search.py:269-335
* ``ghost_stage``        shardann/pipeline.py:158-184
* ``run``                shardann/pipeline.py:270-350 (+ finish :249-267)
* ``reduce_topk``        shardann/pipeline.py:187-196

Parity is pinned by ``tests/test_oracle_golden.py`` against golden vectors
produced by the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

SELECTION = {"full": 0, "direction": 1, "random": 2}
SEED_MODE = {"neighbors": 0, "mixed": 1}


class _Graph(C.Structure):
    _fields_ = [
        ("vectors", C.c_void_p), ("n", C.c_int64), ("d", C.c_int32),
        ("adj", C.c_void_p), ("j", C.c_int32), ("global_ids", C.c_void_p),
        ("direction", C.c_void_p),
    ]


class _Shard(C.Structure):
    _fields_ = [("main", _Graph), ("inter_map", C.c_void_p), ("has_ghost", C.c_int32),
                ("ghost", _Graph)]


class _Params(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("l", C.c_int32), ("m", C.c_int32), ("r", C.c_int32),
        ("max_iter", C.c_int32), ("seed", C.c_uint64), ("selection", C.c_int32),
        ("discard_ratio", C.c_double), ("cooldown_ratio", C.c_double),
        ("ghost_enabled", C.c_int32), ("ghost_max_iter", C.c_int32),
        ("seed_mode", C.c_int32), ("buffer_cap", C.c_int32), ("log_visits", C.c_int32),
        ("metric", C.c_int32), ("forward_count", C.c_int32), ("late_l", C.c_int32),
        ("late_max_iter", C.c_int32),
    ]


class _Pcg(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]


class _Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "iterations", "distance_computations", "total_visits", "nodes_expanded",
        "dgs_skipped", "inserted_total")]


class _Result(C.Structure):
    _fields_ = [("n_out", C.c_int32), ("converged", C.c_int32), ("retained", C.c_int32),
                ("c", _Counters), ("n_visited", C.c_int64)]


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc; no GPU)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _HERE / "liboracle.so"


def lib():
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle.so"
        if not path.exists() or path.stat().st_mtime < (_HERE / "pw_oracle.c").stat().st_mtime:
            build()
        L = C.CDLL(str(path))
        L.orc_last_error.restype = C.c_char_p
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
        L.orc_pcg64_next64.restype = C.c_uint64
        L.orc_pcg64_next32.restype = C.c_uint32
        L.orc_choice.argtypes = [C.POINTER(_Pcg), C.c_int64, C.c_int64, C.c_void_p]
        L.orc_permutation.argtypes = [C.POINTER(_Pcg), C.c_int64, C.c_void_p]
        L.orc_pcg64_seed.argtypes = [C.c_uint64, C.POINTER(_Pcg)]
        L.orc_squared_l2.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_keep_count.argtypes = [C.c_int32, C.c_double]
        L.orc_in_cooldown.argtypes = [C.c_int32, C.c_int32, C.c_double]
        L.orc_search.argtypes = [C.POINTER(_Graph), C.c_void_p, C.POINTER(_Params), C.c_void_p,
                                 C.c_int32, C.POINTER(_Pcg), C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.POINTER(_Result), C.c_void_p, C.c_int64]
        L.orc_ghost_stage.argtypes = [C.POINTER(_Shard), C.c_void_p, C.POINTER(_Params),
                                      C.POINTER(_Pcg), C.POINTER(C.c_int32), C.POINTER(_Counters)]
        L.orc_run.argtypes = [C.POINTER(_Shard), C.c_int32, C.c_void_p, C.c_int64,
                              C.POINTER(_Params), C.c_int32, C.c_int32] + [C.c_void_p] * 7
        L.orc_crc32c_update.restype = C.c_uint32
        L.orc_crc32c_update.argtypes = [C.c_uint32, C.c_void_p, C.c_int64]
        L.orc_reduce_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                      C.c_void_p, C.c_void_p]
        L.orc_run_stage.argtypes = [C.POINTER(_Shard), C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                    C.POINTER(_Params), C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                    C.c_void_p, C.c_int32]
        _LIB = L
    return _LIB


def _err() -> str:
    return lib().orc_last_error().decode()


def _ptr(a):
    return None if a is None else a.ctypes.data


# --------------------------------------------------------------- RNG
def derive_seed(seed: int, *parts: int) -> int:
    arr = (C.c_uint64 * max(1, len(parts)))(*[p & (2**64 - 1) for p in parts])
    return int(lib().orc_derive_seed(seed & (2**64 - 1), arr, len(parts)))


def _pcg_from_state(st: dict) -> _Pcg:
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = 2**64 - 1
    return _Pcg(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))


def _pcg_to_state(g: _Pcg) -> dict:
    return {"bit_generator": "PCG64",
            "state": {"state": (g.state_hi << 64) | g.state_lo, "inc": (g.inc_hi << 64) | g.inc_lo},
            "has_uint32": int(g.has_uint32), "uinteger": int(g.uinteger)}


def pcg64_state(seed64: int) -> dict:
    g = _Pcg()
    lib().orc_pcg64_seed(seed64, C.byref(g))
    return _pcg_to_state(g)


def choice(state: dict, pop: int, size: int):
    g = _pcg_from_state(state)
    out = np.empty(max(size, 1), np.int64)
    if lib().orc_choice(C.byref(g), pop, size, out.ctypes.data):
        raise ValueError(_err())
    return out[:size], _pcg_to_state(g)


def permutation(state: dict, n: int):
    g = _pcg_from_state(state)
    out = np.empty(max(n, 1), np.int64)
    lib().orc_permutation(C.byref(g), n, out.ctypes.data)
    return out[:n], _pcg_to_state(g)


def next64(state: dict, count: int):
    g = _pcg_from_state(state)
    out = [int(lib().orc_pcg64_next64(C.byref(g))) for _ in range(count)]
    return out, _pcg_to_state(g)


# --------------------------------------------------------------- L2 / direction
def squared_l2(points: np.ndarray, q: np.ndarray) -> np.ndarray:
    points = np.ascontiguousarray(points, np.float32)
    q = np.ascontiguousarray(q, np.float32)
    out = np.empty(points.shape[0], np.float32)
    lib().orc_squared_l2(points.ctypes.data, points.shape[0], points.shape[1], q.ctypes.data,
                         out.ctypes.data)
    return out


def keep_count(j: int, discard_ratio: float) -> int:
    return int(lib().orc_keep_count(j, discard_ratio))


def in_cooldown(iteration: int, max_iter: int, cooldown_ratio: float) -> bool:
    return bool(lib().orc_in_cooldown(iteration, max_iter, cooldown_ratio))


# --------------------------------------------------------------- search
def _params(p, ext: dict | None = None) -> _Params:
    """ext: the opt-in path-extension knobs (forward_count, late_l,
    late_max_iter; the GPU's tuning keys of the same names)."""
    ext = ext or {}
    return _Params(int(p.k), int(p.l), int(p.m), int(p.r), int(p.max_iter),
                   int(p.seed) & (2**64 - 1), SELECTION[p.selection], float(p.discard_ratio),
                   float(p.cooldown_ratio), int(bool(p.ghost_enabled)), int(p.ghost_max_iter),
                   SEED_MODE[p.seed_mode], int(p.buffer_cap or 0), int(bool(p.log_visits)),
                   {"l2": 0, "ip": 1}[getattr(p, "metric", "l2")], int(ext.get("forward_count", 0)),
                   int(ext.get("late_l", 0)), int(ext.get("late_max_iter", 0)))


class _Keep:
    """Holds numpy arrays alive while C structs point into them."""

    def __init__(self):
        self.refs = []

    def arr(self, a, dtype):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype)
        self.refs.append(a)
        return a


def _graph(keep: _Keep, vectors, adj, global_ids, direction=None) -> _Graph:
    v = keep.arr(vectors, np.float32)
    a = keep.arr(adj, np.int32)
    g = keep.arr(global_ids, np.int32)
    dr = keep.arr(direction, np.uint32)
    j = a.shape[1] if a.ndim == 2 else 0
    return _Graph(v.ctypes.data, v.shape[0], v.shape[1], a.ctypes.data, j, g.ctypes.data,
                  _ptr(dr))


def _shard(keep: _Keep, ctx) -> _Shard:
    main = _graph(keep, ctx.vectors, ctx.adj, ctx.global_ids, getattr(ctx, "direction", None))
    inter = keep.arr(getattr(ctx, "inter_map", None), np.int32)
    gh = getattr(ctx, "ghost", None)
    if gh is not None:
        ghost = _graph(keep, gh.vectors, gh.adj, gh.parent_ids)
        return _Shard(main, _ptr(inter), 1, ghost)
    return _Shard(main, _ptr(inter), 0, _Graph())


def search(query, ctx, params, seeds=(), *, rng_state: dict, visit_cap: int = 1 << 20):
    """search.py:269 on one context; returns (dict, advanced rng state)."""
    keep = _Keep()
    g = _graph(keep, ctx.vectors, ctx.adj, ctx.global_ids, getattr(ctx, "direction", None))
    q = keep.arr(query, np.float32)
    s = keep.arr(np.asarray([int(x) for x in seeds], np.int64).reshape(-1), np.int64)
    p = _params(params)
    pcg = _pcg_from_state(rng_state)
    k = int(params.k)
    ids = np.empty(k, np.int32)
    dists = np.empty(k, np.float32)
    loc = np.empty(k, np.int32)
    log = np.empty(visit_cap if params.log_visits else 1, np.int32)
    res = _Result()
    rc = lib().orc_search(C.byref(g), q.ctypes.data, C.byref(p), s.ctypes.data, len(s),
                          C.byref(pcg), ids.ctypes.data, dists.ctypes.data, loc.ctypes.data,
                          C.byref(res), log.ctypes.data, len(log))
    if rc:
        raise ValueError(_err())
    n = res.n_out
    c = res.c
    out = dict(ids=ids[:n].copy(), dists=dists[:n].copy(), local_ids=loc[:n].copy(),
               converged=bool(res.converged), retained=int(res.retained),
               counters=dict(iterations=c.iterations, distance_computations=c.distance_computations,
                             total_visits=c.total_visits, nodes_expanded=c.nodes_expanded,
                             dgs_skipped=c.dgs_skipped, inserted_total=c.inserted_total),
               visited_ids=log[:res.n_visited].copy() if params.log_visits else None)
    return out, _pcg_to_state(pcg)


def ghost_stage(query, ctx, params, *, rng_state: dict):
    keep = _Keep()
    sh = _shard(keep, ctx)
    q = keep.arr(query, np.float32)
    p = _params(params)
    pcg = _pcg_from_state(rng_state)
    entry = C.c_int32()
    cnt = _Counters()
    if lib().orc_ghost_stage(C.byref(sh), q.ctypes.data, C.byref(p), C.byref(pcg),
                             C.byref(entry), C.byref(cnt)):
        raise ValueError(_err())
    return int(entry.value), dict(iterations=cnt.iterations,
                                  distance_computations=cnt.distance_computations,
                                  total_visits=cnt.total_visits), _pcg_to_state(pcg)


STAT_I32 = ("iterations", "ghost_iterations", "retained", "converged")
STAT_I64 = ("distance_computations", "total_visits", "inserted", "dgs_skipped")


def run(queries: np.ndarray, contexts, params, mode: str, threads: int = 0, ext: dict | None = None) -> dict:
    """pipeline.py run_sharded_baseline (mode='baseline') / run_pipelined.
    ext: opt-in path-extension knobs (not the reference; see _params)."""
    keep = _Keep()
    n = len(contexts)
    arr = (_Shard * n)(*[_shard(keep, c) for c in contexts])
    q = keep.arr(queries, np.float32)
    nq = q.shape[0]
    k = int(params.k)
    p = _params(params, ext)
    shard_ids = np.empty((nq, n, k), np.int32)
    shard_dists = np.empty((nq, n, k), np.float32)
    final_ids = np.empty((nq, k), np.int32)
    final_dists = np.empty((nq, k), np.float32)
    s32 = np.empty((n, 4, nq), np.int32)
    s64 = np.empty((n, 4, nq), np.int64)
    comm = np.empty((n, n), np.int64)
    rc = lib().orc_run(arr, n, q.ctypes.data, nq, C.byref(p), 0 if mode == "baseline" else 1,
                       int(threads), shard_ids.ctypes.data, shard_dists.ctypes.data,
                       final_ids.ctypes.data, final_dists.ctypes.data, s32.ctypes.data,
                       s64.ctypes.data, comm.ctypes.data)
    if rc:
        raise ValueError(_err())
    stages = []
    for s in range(n):
        st = {name: s32[s, i].copy() for i, name in enumerate(STAT_I32)}
        st.update({name: s64[s, i].copy() for i, name in enumerate(STAT_I64)})
        st["converged"] = st["converged"].astype(bool)
        stages.append(st)
    return dict(shard_ids=shard_ids, shard_dists=shard_dists, final_ids=final_ids,
                final_dists=final_dists, stages=stages, comm_stage_bytes=comm)


def crc32c(data) -> int:
    """_crc32c.py:98-130 crc32c (serial definition, _crc32c.py:17-37)."""
    buf = np.ascontiguousarray(np.frombuffer(data, np.uint8) if isinstance(data, (bytes, bytearray))
                               else np.asarray(data).view(np.uint8).ravel())
    raw = lib().orc_crc32c_update(0xFFFFFFFF, buf.ctypes.data if buf.size else None, buf.size)
    return (~raw) & 0xFFFFFFFF


def reduce_topk(ids, dists, k: int):
    ids = np.ascontiguousarray(np.asarray(ids).ravel(), np.int32)
    dists = np.ascontiguousarray(np.asarray(dists).ravel(), np.float32)
    oi = np.empty(max(k, 1), np.int32)
    od = np.empty(max(k, 1), np.float32)
    rc = lib().orc_reduce_topk(ids.ctypes.data, dists.ctypes.data, ids.size, k, oi.ctypes.data,
                               od.ctypes.data)
    if rc < 0:
        raise ValueError(_err())
    return oi[:rc], od[:rc]


def run_stage(ctx, queries: np.ndarray, q0: int, n: int, params, stage: int, entries_in, forward_out,
              shard_ids, shard_dists, col: int, stats_i32, stats_i64, threads: int = 0) -> None:
    """One stage of one shard on the CPU (mirror of pw_search_stage); the
    output arrays are numpy arrays updated in place."""
    keep = _Keep()
    sh = _shard(keep, ctx)
    q = keep.arr(queries, np.float32)
    p = _params(params)
    rc = lib().orc_run_stage(C.byref(sh), q.ctypes.data, q.shape[0], q0, n, C.byref(p), stage,
                             _ptr(entries_in), _ptr(forward_out), shard_ids.ctypes.data,
                             shard_dists.ctypes.data, shard_ids.shape[1], col,
                             stats_i32.ctypes.data, stats_i64.ctypes.data, int(threads))
    if rc:
        raise ValueError(_err())
