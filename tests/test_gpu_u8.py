"""uint8 vector rows (BASELINE C3, SIFT-shaped bvecs).  The reference keeps
float32 rows (data.py:36 upcasts); byte-valued rows are stored as uint8 on
the device and rebuilt exactly as float(b), so every result must be
bit-identical to the oracle on the float32 upcast."""

import numpy as np
import pytest

import oracle
import paper_2507_17094_b200 as pw
from golden_util import assert_run_equal, assert_run_equal_lossy, oracle_dict, result_dict
from index_util import clustered, make_contexts
from paper_2507_17094_b200.search import SearchParams, byte_rows, device_shard


def byte_data(n, d, seed):
    x = clustered(n, d, 256, 0.08, seed=seed)
    return np.clip(np.rint(255.0 * x), 0, 255).astype(np.float32)


ARMS = [
    dict(k=10, l=64, m=64, r=8, max_iter=64, seed=1),
    dict(k=10, l=128, m=64, r=8, max_iter=64, seed=2, selection="direction", discard_ratio=0.5,
         cooldown_ratio=0.3, ghost_enabled=True, ghost_max_iter=8),
    dict(k=10, l=96, m=64, r=4, max_iter=10, seed=3, selection="random", discard_ratio=0.5,
         seed_mode="mixed", ghost_enabled=True),
]


def test_byte_rows_detection():
    assert byte_rows(np.zeros((3, 8), np.float32))
    assert byte_rows(np.full((3, 8), 255, np.float32))
    assert not byte_rows(np.full((3, 8), 255.5, np.float32))
    assert not byte_rows(np.full((3, 8), 256, np.float32))
    assert not byte_rows(np.full((3, 8), -1, np.float32))
    assert not byte_rows(np.zeros((3, 6), np.float32))  # d % 4 != 0
    assert byte_rows(np.zeros((3, 8), np.uint8))


@pytest.fixture(scope="module")
def u8sets():
    out = {}
    # 96 / 128: specialised uint8 kernels; 64, 100: the generic uint8 kernel
    for d, n, nq, shards in ((128, 12000, 300, 2), (96, 12000, 300, 3), (64, 6000, 200, 2),
                             (100, 6000, 200, 2)):
        x = byte_data(n + nq, d, seed=d + 7)
        out[d] = (np.ascontiguousarray(x[n:]), make_contexts(x[:n], shards, 32, seed=d))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("d", [128, 96, 64, 100])
@pytest.mark.parametrize("arm", range(len(ARMS)))
@pytest.mark.parametrize("mode", ["baseline", "pipelined"])
def test_u8_rows_match_oracle(u8sets, d, arm, mode):
    queries, ctxs = u8sets[d]
    params = SearchParams(**ARMS[arm])
    runner = pw.run_sharded_baseline if mode == "baseline" else pw.run_pipelined
    got = result_dict(runner(pw.Dataset(queries), None, None, params, contexts=ctxs))
    assert all(device_shard(c).dtype == "u8" for c in ctxs)
    want = oracle_dict(oracle.run(queries, ctxs, params, mode))
    assert_run_equal(got, want, f"u8 d={d} arm={arm} {mode}")
    lossy = result_dict(runner(pw.Dataset(queries), None, None, params, contexts=ctxs,
                               tuning={"flags": 2}))
    assert_run_equal_lossy(lossy, want, f"u8 lossy d={d} arm={arm} {mode}")


@pytest.mark.gpu
def test_u8_squared_l2_primitive():
    import torch

    from paper_2507_17094_b200.search import ShardContext

    lib = pw._abi.load()
    rs = np.random.default_rng(5)
    for d in (8, 96, 128, 200, 964):
        x = rs.integers(0, 256, size=(300, d)).astype(np.float32)
        q = (rs.random(d, dtype=np.float32) * 255).astype(np.float32)
        ctx = ShardContext(vectors=x, adj=np.zeros((300, 0), np.int32),
                           global_ids=np.arange(300, dtype=np.int32))
        dev = device_shard(ctx)
        assert dev.dtype == "u8"
        ids = torch.arange(300, dtype=torch.int32, device="cuda")
        out = torch.empty(300, dtype=torch.float32, device="cuda")
        tq = torch.from_numpy(q).cuda()
        pw._abi.check(lib.pw_squared_l2_rows(dev.handle, ids.data_ptr(), 300, tq.data_ptr(),
                                             out.data_ptr(), None))
        torch.cuda.synchronize()
        want = oracle.squared_l2(x, q)
        assert np.array_equal(out.cpu().numpy(), want), d


@pytest.mark.gpu
@pytest.mark.parametrize("d", [128, 96])
@pytest.mark.parametrize("shift", ["fraction", "out_of_range", "mixed"])
def test_u8_rows_nonintegral_queries_match_oracle(u8sets, d, shift):
    """Byte rows against queries that are NOT integers in [0, 255]: K1 must take
    the float path (pw_row4_u8) instead of the exact DP4A integer path, per
    query; a batch mixing both kinds exercises the per-task switch."""
    queries, ctxs = u8sets[d]
    q = queries.copy()
    if shift == "fraction":
        q += np.float32(0.25)
    elif shift == "out_of_range":
        q[:, 0] = 300.0
    else:
        q[::2] += np.float32(0.5)
    for arm in (0, 1):
        params = SearchParams(**ARMS[arm])
        for mode, runner in (("baseline", pw.run_sharded_baseline), ("pipelined", pw.run_pipelined)):
            got = result_dict(runner(pw.Dataset(q), None, None, params, contexts=ctxs))
            want = oracle_dict(oracle.run(q, ctxs, params, mode))
            assert_run_equal(got, want, f"u8 {shift} d={d} arm={arm} {mode}")


@pytest.mark.gpu
@pytest.mark.parametrize("d", [128, 96])
@pytest.mark.parametrize("arm", range(len(ARMS)))
@pytest.mark.parametrize("flags", [8, 10])
def test_u8_rows_tma_gather4_match_oracle(u8sets, d, arm, flags):
    """Scoring rows by TMA tile::gather4 (tuning flag 8) on uint8 rows."""
    queries, ctxs = u8sets[d]
    params = SearchParams(**ARMS[arm])
    got = result_dict(pw.run_pipelined(pw.Dataset(queries), None, None, params, contexts=ctxs,
                                       tuning={"flags": flags}))
    want = oracle_dict(oracle.run(queries, ctxs, params, "pipelined"))
    (assert_run_equal_lossy if flags & 2 else assert_run_equal)(got, want, f"u8 tma d={d} arm={arm}")
