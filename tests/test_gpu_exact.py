"""Exact GPU index build (exact.build_index) and exact kNN
ground truth (exact.exact_knn_batch, f2) against what the REFERENCE built for
the golden fixtures (tests/golden/make_golden.py ran shardann.build_index and
shardann.exact_knn_batch): every array must be equal."""

import numpy as np
import pytest

import oracle
from golden_util import GOLDEN
from paper_2507_17094_b200 import exact

pytestmark = pytest.mark.gpu

FIXTURES = {  # make_golden.py build_index arguments
    "small": dict(n_shards=4, j=16, seed=5, rho=0.05, ghost_degree=8),
    "sift128": dict(n_shards=2, j=32, seed=0, rho=0.02, ghost_degree=16),
}


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_build_index_matches_reference(name):
    _check_build(name)


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_build_index_tensor_core_screen_matches_reference(name, monkeypatch):
    """Every screen through K4 (tcgen05 TF32 + certification + FP32 redo of
    uncertified rows): the reference's indexes all the same."""
    monkeypatch.setattr(exact, "TC_MIN_PAIRS", 0)
    _check_build(name)


def _check_build(name):
    z = np.load(GOLDEN / f"{name}.npz")
    kw = FIXTURES[name]
    index, report = exact.build_index(z["base"], kw["n_shards"], kw["j"], kw["seed"], rho=kw["rho"],
                                      ghost_degree=kw["ghost_degree"])
    assert index.n_shards == int(z["n_shards"]) and index.d == z["base"].shape[1]
    assert report.total > 0
    for s, pack in enumerate(index.shards):
        for field in ("global_ids", "adj", "inter_map", "ghost_ids", "ghost_adj"):
            want = z[f"s{s}_{field}"]
            got = getattr(pack, field)
            assert got is not None and got.shape == want.shape, (name, s, field)
            assert np.array_equal(got, want), (name, s, field, np.argwhere(got != want)[:5])
        d = pack.direction
        if f"s{s}_direction" in z:
            assert np.array_equal(d, z[f"s{s}_direction"]), (name, s, "direction")
        else:
            assert np.uint64(d.astype(np.uint64).sum()) == z[f"s{s}_direction_sum"]
            assert np.uint32(np.bitwise_xor.reduce(d.ravel())) == z[f"s{s}_direction_xor"]


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_exact_knn_matches_reference_truth(name):
    z = np.load(GOLDEN / f"{name}.npz")
    if "truth_ids" not in z.files:
        pytest.skip(f"{name}.npz carries no reference ground truth")
    ids, dists = exact.exact_knn_batch(z["base"], z["queries"], 10)
    assert np.array_equal(ids, z["truth_ids"])
    assert np.array_equal(dists, z["truth_dists"])


@pytest.mark.parametrize("d", [1, 7, 16, 96, 128, 200, 960])
def test_l2_pairs_bit_exact(d):
    import torch

    rs = np.random.default_rng(d)
    a = rs.standard_normal((300, d), dtype=np.float32)
    b = rs.standard_normal((500, d), dtype=np.float32) * np.float32(3.0)
    ia = rs.integers(0, 300, 4001)
    ib = rs.integers(0, 500, 4001)
    got = exact.l2_pairs(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                         torch.from_numpy(ia).cuda(), torch.from_numpy(ib).cuda()).cpu().numpy()
    want = np.array([oracle.squared_l2(b[ib[t]][None, :], a[ia[t]])[0] for t in range(len(ia))], np.float32)
    assert np.array_equal(got, want)


def test_build_errors():
    x = np.random.default_rng(0).standard_normal((40, 8), dtype=np.float32)
    with pytest.raises(ValueError, match="need 1 <= N <= n"):
        exact.build_index(x, 0, 4, 1)
    with pytest.raises(ValueError, match="need 0 <= j < n_local"):
        exact.build_index(x, 2, 20, 1)
    import torch

    with pytest.raises(ValueError, match="too small for out-degree"):
        exact.build_ghost_index(torch.from_numpy(x).cuda(), 0.1, 8, 1)


@pytest.mark.parametrize("d,n,nq,self_ex,dup", [(96, 40000, 3000, True, False), (128, 20000, 2000, False, False),
                                                (100, 12000, 1000, True, False), (96, 30000, 2000, True, True),
                                                (16, 40, 40, True, False), (200, 30000, 2000, True, False),
                                                (200, 12000, 1000, False, True), (960, 6000, 600, True, False)])
def test_tensor_core_screen_topk_equals_fp32_screen(d, n, nq, self_ex, dup):
    """exact_topk through K4 (certified, redo of the rest) == through the FP32
    screen, ids and bit-exact distances; with duplicate rows (exact distance
    ties, broken by id) and with fewer base rows than candidates."""
    import torch

    from paper_2507_17094_b200 import builder

    x = builder.gen_latent(n, d, 16, 1, 1.0, 0.05, d + n, device="cuda")
    if dup:
        x[1::3] = x[0::3][: x[1::3].shape[0]]  # every third row duplicated
    q = x[:nq].contiguous() if self_ex else builder.gen_latent(nq, d, 16, 1, 1.0, 0.05, 99, device="cuda")
    k = min(32, n - 1)
    st = {}
    a_ids, a_sq = exact.exact_topk(x, q, k, exclude_self=self_ex, screen="tc", stats=st)
    b_ids, b_sq = exact.exact_topk(x, q, k, exclude_self=self_ex, screen="fp32")
    assert torch.equal(a_ids, b_ids), st
    assert torch.equal(a_sq, b_sq)
    assert st["certified"] + st["redone"] == nq
    if n >= 1000:  # the screen does the work: most rows need no FP32 redo
        assert st["certified"] >= 0.9 * nq, st


def test_tensor_core_screen_shape_limits():
    """d = 200 and 960 do not leave room for K4's resident query block: K4
    streams it per K atom (its values equal the resident path's on the same
    columns); rows that are not 16-byte multiples or lists past 64 raise."""
    import torch

    from paper_2507_17094_b200 import builder

    x = builder.gen_latent(3000, 200, 16, 1, 1.0, 0.05, 5, device="cuda")
    ids, vals, _ = exact.knn_screen_tc(x, x[:300].contiguous(), 64)
    # the screened values are TF32 approximations of |x|^2 - 2 q.x
    ref = (x * x).sum(1)[ids.clamp(min=0)] - 2 * (x[:300, None, :] * x[ids.clamp(min=0)]).sum(-1)
    assert (ids >= 0).all() and torch.allclose(vals, ref, rtol=0, atol=2e-2 * float(ref.abs().max()))
    with pytest.raises(ValueError, match="unsupported"):
        exact.knn_screen_tc(x, x[:10].contiguous(), 65)
    with pytest.raises(ValueError, match="unsupported"):
        y = builder.gen_latent(300, 30, 16, 1, 1.0, 0.05, 5, device="cuda")
        exact.knn_screen_tc(y, y[:10].contiguous(), 16)
    a, _ = exact.exact_topk(x, x[:50].contiguous(), 10, screen="auto")
    b, _ = exact.exact_topk(x, x[:50].contiguous(), 10, screen="fp32")
    assert torch.equal(a, b)
