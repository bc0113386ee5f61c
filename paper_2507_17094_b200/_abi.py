"""ctypes binding of libpwb200.so (the C ABI declared in include/pw_b200.h).

The CUDA library is the only compute path: if it is missing or no CUDA device
is visible, every entry point raises instead of falling back to the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["PW_LIB"]) if os.environ.get("PW_LIB") else _PKG / "libpwb200.so"

PW_OK, PW_EINVAL, PW_ENOMEM, PW_ECUDA = 0, -1, -2, -3
SELECTION = {"full": 0, "direction": 1, "random": 2}
SEED_MODE = {"neighbors": 0, "mixed": 1}
MODE = {"baseline": 0, "pipelined": 1}


class Params(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("l", C.c_int32), ("m", C.c_int32), ("r", C.c_int32),
        ("max_iter", C.c_int32), ("seed", C.c_uint64), ("selection", C.c_int32),
        ("discard_ratio", C.c_double), ("cooldown_ratio", C.c_double),
        ("ghost_enabled", C.c_int32), ("ghost_max_iter", C.c_int32), ("seed_mode", C.c_int32),
        ("buffer_cap", C.c_int32), ("log_visits", C.c_int32), ("metric", C.c_int32),
    ]


class Tuning(C.Structure):
    _fields_ = [("visited_slots", C.c_int32), ("stage_rows", C.c_int32),
                ("warps_per_sm", C.c_int32), ("row_copy", C.c_int32), ("flags", C.c_int32),
                ("forward_count", C.c_int32), ("late_l", C.c_int32), ("late_max_iter", C.c_int32)]


class ShardDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("d", C.c_int32), ("j", C.c_int32), ("dtype", C.c_int32),
        ("vectors", C.c_void_p), ("adj", C.c_void_p), ("global_ids", C.c_void_p),
        ("direction", C.c_void_p), ("inter_map", C.c_void_p), ("ghost_n", C.c_int64),
        ("ghost_j", C.c_int32), ("ghost_ids", C.c_void_p), ("ghost_adj", C.c_void_p),
        ("on_device", C.c_int32),
    ]


class Rng(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]


class SearchOut(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("distance_computations", C.c_int64),
        ("total_visits", C.c_int64), ("nodes_expanded", C.c_int64), ("dgs_skipped", C.c_int64),
        ("inserted_total", C.c_int64), ("converged", C.c_int32), ("retained", C.c_int32),
        ("n_out", C.c_int32), ("pad_", C.c_int32), ("n_visited", C.c_int64),
    ]


EXPORTS = {
    "pw_last_error": (C.c_char_p, []),
    "pw_version": (C.c_char_p, []),
    "pw_launch_count": (C.c_int64, []),
    "pw_shard_create": (C.c_int, [C.POINTER(ShardDesc), C.POINTER(C.c_void_p)]),
    "pw_shard_destroy": (C.c_int, [C.c_void_p]),
    "pw_shard_bytes": (C.c_int64, [C.c_void_p]),
    "pw_search_one": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Params), C.c_void_p, C.c_void_p,
                                C.c_int32, C.POINTER(Rng), C.c_void_p, C.c_void_p, C.c_void_p,
                                C.POINTER(SearchOut), C.c_void_p, C.c_int64]),
    "pw_search_stage": (C.c_int, [C.c_void_p, C.POINTER(Params), C.POINTER(Tuning), C.c_void_p,
                                  C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_int64, C.c_void_p]),
    "pw_init_outputs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_int64, C.c_void_p]),
    "pw_reduce_topk": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pw_run": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Params), C.POINTER(Tuning), C.c_void_p,
                         C.c_int64, C.c_int32] + [C.c_void_p] * 7),
    "pw_run_device": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Params), C.POINTER(Tuning),
                                C.c_void_p, C.c_int64, C.c_int32] + [C.c_void_p] * 9),
    "pw_squared_l2_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "pw_launch_config": (C.c_int, [C.c_void_p, C.POINTER(Params), C.POINTER(Tuning), C.c_void_p]),
    "pw_phase_cycles": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "pw_search_dataflow": (C.c_int, [C.c_void_p, C.POINTER(Params), C.POINTER(Tuning), C.c_void_p,
                                     C.c_int64, C.c_int32, C.c_int32, C.c_uint32, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_int32, C.c_void_p]),
    "pw_shard_check": (C.c_int, [C.c_void_p]),
    "pw_shard_validate_inter": (C.c_int, [C.c_void_p, C.c_int64]),
    "pw_signal": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p]),
    "pw_wait": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "pw_l2_pairs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_void_p, C.c_void_p]),
    "pw_knn_screen": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pw_gather_probe": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                  C.c_void_p]),
    "pw_dev_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    "pw_dev_free": (C.c_int, [C.c_void_p]),
    "pw_ipc_get": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pw_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pw_ipc_close": (C.c_int, [C.c_void_p]),
    "pw_crc32c": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_uint32)]),
    "pw_crc32c_combine": (C.c_int, [C.c_uint32, C.c_uint32, C.c_int64, C.POINTER(C.c_uint32)]),
    "pw_crc32c_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
}

OPTIONAL = {"pw_init_outputs", "pw_shard_validate_inter", "pw_signal", "pw_wait", "pw_phase_cycles", "pw_launch_config", "pw_search_dataflow", "pw_shard_check", "pw_l2_pairs", "pw_knn_screen", "pw_gather_probe", "pw_dev_alloc", "pw_dev_free",
            "pw_ipc_get", "pw_ipc_open", "pw_ipc_close"}
_LIB = None


def load(require_device: bool = True):
    """Load libpwb200.so; raise loudly when the native path is unavailable."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA extension is the only compute path; there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                if name in OPTIONAL:  # older builds loaded via PW_LIB for A/B runs
                    continue
                raise RuntimeError(f"{LIB_PATH} lacks {name}: rebuild it")
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device visible: the B200 search path has no CPU fallback")
    return _LIB


def check(rc: int) -> None:
    if rc == PW_OK:
        return
    msg = _LIB.pw_last_error().decode()
    if rc == PW_EINVAL:
        raise ValueError(msg)
    if rc == PW_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def params_struct(p) -> Params:
    if p.selection not in SELECTION:
        raise ValueError(f"selection must be one of {tuple(SELECTION)}")
    if p.seed_mode not in SEED_MODE:
        raise ValueError(f"seed_mode must be one of {tuple(SEED_MODE)}")
    return Params(int(p.k), int(p.l), int(p.m), int(p.r), int(p.max_iter),
                  int(p.seed) & (2**64 - 1), SELECTION[p.selection], float(p.discard_ratio),
                  float(p.cooldown_ratio), int(bool(p.ghost_enabled)), int(p.ghost_max_iter),
                  SEED_MODE[p.seed_mode], int(p.buffer_cap or 0), int(bool(p.log_visits)),
                  METRIC[getattr(p, "metric", "l2")])


METRIC = {"l2": 0, "ip": 1}


def tuning_struct(t) -> Tuning:
    if t is None:
        return Tuning(0, 0, 0, 0, 0, 0, 0, 0)
    return Tuning(int(t.get("visited_slots", 0)), int(t.get("stage_rows", 0)),
                  int(t.get("warps_per_sm", 0)), int(t.get("row_copy", 0)), int(t.get("flags", 0)),
                  int(t.get("forward_count", 0)), int(t.get("late_l", 0)), int(t.get("late_max_iter", 0)))


def forward_count(t) -> int:
    """Entries forwarded per query (tuning "forward_count", default 1)."""
    return max(1, int((t or {}).get("forward_count", 0) or 1))


def launch_config(shard_handle, params, tuning=None) -> dict:
    """K1 launch configuration for a shard/params/tuning (no launch)."""
    lib = load()
    out = (C.c_int32 * 6)()
    p = params_struct(params)
    t = tuning_struct(tuning)
    check(lib.pw_launch_config(shard_handle, C.byref(p), C.byref(t), out))
    return dict(warps_per_sm=out[0], smem_per_warp=out[1], visited_slots=out[2], stage_rows=out[3],
                specialised_d=out[4], blocks=out[5])


def result_block(q: int, n: int, k: int, pinned: bool = False) -> dict:
    """pw_run's six output arrays as views into one allocation in the result
    block layout of include/pw_b200.h (shard_ids | shard_dists | final_ids |
    final_dists | stats_i32 | stats_i64, each at the previous start + its
    size rounded up to 256 bytes), so pw_run copies them in one transfer.
    `pinned`: page-locked (torch) memory, DMA straight into it."""
    import numpy as np

    specs = (("shard_ids", (q, n, k), np.int32), ("shard_dists", (q, n, k), np.float32),
             ("final_ids", (q, k), np.int32), ("final_dists", (q, k), np.float32),
             ("s32", (n, 4, q), np.int32), ("s64", (n, 6, q), np.int64))
    offs, total = [], 0
    for _, shape, dt in specs:
        offs.append(total)
        nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
        total += (nbytes + 255) // 256 * 256
    if pinned:
        import torch

        raw = torch.empty(total + 256, dtype=torch.uint8, pin_memory=True).numpy()
    else:
        raw = np.empty(total + 256, np.uint8)
    base = (-raw.ctypes.data) % 256  # 256-byte aligned start (not required, but tidy)
    out = {}
    for (name, shape, dt), o in zip(specs, offs):
        nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
        out[name] = raw[base + o:base + o + nbytes].view(dt).reshape(shape)
    out["_raw"] = raw  # keeps the allocation alive with the views
    return out
