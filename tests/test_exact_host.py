"""Host-side halves of the exact GPU index build (exact.py) against the
indexes the reference built for the golden fixtures: the partition and the
ghost sample come from the reference's numpy streams (no device needed)."""

import numpy as np
import pytest

from golden_util import GOLDEN
from paper_2507_17094_b200 import exact
from paper_2507_17094_b200.rng import TAG_GHOST_SAMPLE, stream

FIXTURES = {  # make_golden.py build_index arguments
    "small": dict(n_shards=4, j=16, seed=5, rho=0.05, ghost_degree=8),
    "sift128": dict(n_shards=2, j=32, seed=0, rho=0.02, ghost_degree=16),
}


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_partition_and_ghost_sample_match_reference(name):
    z = np.load(GOLDEN / f"{name}.npz")
    kw = FIXTURES[name]
    rows = exact.partition_rows(z["base"].shape[0], kw["n_shards"], kw["seed"])
    for s, r in enumerate(rows):
        assert np.array_equal(r.astype(np.int32), z[f"s{s}_global_ids"])
        g = exact.ghost_count(len(r), kw["rho"])
        ids = np.sort(stream(kw["seed"], TAG_GHOST_SAMPLE, s).choice(len(r), size=g, replace=False))
        assert np.array_equal(ids.astype(np.int32), z[f"s{s}_ghost_ids"])


def test_ghost_count_epsilon():
    assert exact.ghost_count(10000, 0.01) == 100   # 0.01 * 10000 = 100.00000000000001
    assert exact.ghost_count(1001, 0.01) == 11


def test_partition_validation():
    with pytest.raises(ValueError, match="need 1 <= N <= n"):
        exact.partition_rows(3, 4, 0)
