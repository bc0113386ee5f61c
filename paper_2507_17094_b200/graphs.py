"""Index types of the reference (shardann/graphs.py:189-215).

The search path consumes these; building them is the reference's offline
``build_index`` (graphs.py:237-299), out of this path's scope.  Indexes built
by the reference (``shardann.Index``) or by ``paper_2507_17094_b200.builder``
are interchangeable: only the attribute names below are read.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def words_per_vector(d: int) -> int:
    """direction.py:23-25: packed uint32 words for d sign bits."""
    return (d + 31) // 32


@dataclass(frozen=True)
class ShardPack:
    """Per-shard bundle (graphs.py:189-202); vectors live in the dataset."""

    global_ids: np.ndarray            # (n_local,) int32
    adj: np.ndarray                   # (n_local, j) int32
    inter_map: np.ndarray | None      # (n_local,) int32, None for N == 1
    ghost_ids: np.ndarray | None      # (g,) int32
    ghost_adj: np.ndarray | None      # (g, j_g) int32
    direction: np.ndarray | None      # (n_local, j, W) uint32

    @property
    def n_local(self) -> int:
        return self.global_ids.shape[0]


@dataclass(frozen=True)
class Index:
    """All per-shard structures for one dataset (graphs.py:205-215)."""

    d: int
    n_total: int
    shards: list

    @property
    def n_shards(self) -> int:
        return len(self.shards)
