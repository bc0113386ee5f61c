"""Helpers for the dataflow-ring tests: ShardContext -> TensorShard, and a
device run laid out like golden_util.oracle_dict (comm excluded)."""

from __future__ import annotations

import numpy as np

from golden_util import STAT_FIELDS


def tensor_shard(ctx):
    import torch

    from paper_2507_17094_b200 import device as dv

    def t(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()

    d = getattr(ctx, "direction", None)
    gh = getattr(ctx, "ghost", None)
    return dv.TensorShard(t(ctx.vectors), t(ctx.adj), t(ctx.global_ids),
                          None if d is None else t(np.asarray(d).view(np.int32)),
                          t(getattr(ctx, "inter_map", None)),
                          None if gh is None else t(gh.parent_ids), None if gh is None else t(gh.adj))


def run_dict(shard_ids, shard_dists, final_ids, final_dists, s32, s64) -> dict:
    from paper_2507_17094_b200.device import STAT_I32, STAT_I64

    out = dict(final_ids=np.asarray(final_ids), final_dists=np.asarray(final_dists),
               shard_ids=np.asarray(shard_ids), shard_dists=np.asarray(shard_dists))
    s32, s64 = np.asarray(s32), np.asarray(s64)
    for f in STAT_FIELDS:
        if f in STAT_I32:
            out[f] = s32[:, STAT_I32.index(f)]
        else:
            key = "inserted" if f == "inserted" else f
            out[f] = s64[:, STAT_I64.index(key)]
    return out


def assert_same(got: dict, want: dict, what: str, lossy: bool = False) -> None:
    for key in ("final_ids", "final_dists", "shard_ids", "shard_dists"):
        a, b = got[key], want[key]
        assert a.shape == b.shape, (what, key, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{what}: {key} differs at {bad.tolist()}")
    for f in STAT_FIELDS:
        a, b = np.asarray(got[f]).astype(np.int64), np.asarray(want[f]).astype(np.int64)
        if lossy and f == "distance_computations":
            assert np.all(a >= b), (what, f)
            continue
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{what}: stat {f} differs at {bad.tolist()}")
