"""Test infrastructure: the reference's synthetic generator (shardann
data.py:159-176), restated so the acceptance KATs can rebuild the
reference's datasets bit for bit (checked against the reference's own
fixture in test_acceptance_ds2.py).  Not part of the product package: the
bench makes its 10M+ inputs on the device (builder.gen_latent)."""

from __future__ import annotations

import numpy as np

from paper_2507_17094_b200.data import Dataset
from paper_2507_17094_b200.rng import TAG_GEN, stream


def gen_synthetic(n: int, d: int, n_clusters: int, spread: float, seed: int) -> Dataset:
    """Gaussian blobs around uniform [0, 1)^d centres, point i in cluster
    i mod n_clusters; both draws come from the (seed, TAG_GEN) PCG64 stream in
    the reference's order (centres first, then the float32 normals)."""
    if not (1 <= n_clusters <= n):
        raise ValueError(f"need n >= n_clusters >= 1, got n={n}, n_clusters={n_clusters}")
    if d < 1:
        raise ValueError(f"dimension must be >= 1, got {d}")
    if not spread > 0:
        raise ValueError(f"spread must be > 0, got {spread}")
    g = stream(seed, TAG_GEN)
    centres = g.random((n_clusters, d), dtype=np.float32)
    x = g.standard_normal((n, d), dtype=np.float32) * np.float32(spread)
    x += centres[np.arange(n) % n_clusters]
    return Dataset(x)
