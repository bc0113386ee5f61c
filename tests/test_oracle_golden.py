"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

CPU-only: these run in the build container and on the GPU box alike.
"""

import numpy as np
import pytest

import oracle
from golden_util import GOLDEN, assert_run_equal, expected, load, oracle_dict, sift_cases, small_cases
from paper_2507_17094_b200 import rng as prng
from paper_2507_17094_b200.search import SearchParams


def test_derive_seed_golden():
    z = np.load(GOLDEN / "rng.npz")
    for parts, want in zip(z["ds_parts"], z["ds_out"]):
        a, b, c, d = (int(x) for x in parts)
        assert oracle.derive_seed(a, b, c, d) == int(want)
        assert prng.derive_seed(a, b, c, d) == int(want)


def test_pcg64_seeding_golden():
    z = np.load(GOLDEN / "rng.npz")
    for sd, st in zip(z["seeds"], z["states"]):
        got = oracle.pcg64_state(int(sd))
        assert got["state"]["state"] == (int(st[0]) << 64) | int(st[1])
        assert got["state"]["inc"] == (int(st[2]) << 64) | int(st[3])


def test_choice_golden():
    z = np.load(GOLDEN / "rng.npz")
    for case, want in zip(z["choice_cases"], z["choice_out"]):
        sd, pop, size, s_hi, s_lo, has32, u32 = (int(x) for x in case)
        got, st = oracle.choice(oracle.pcg64_state(sd), pop, size)
        assert got.tolist() == want[:size].tolist(), (pop, size)
        assert st["state"]["state"] == (s_hi << 64) | s_lo
        assert st["has_uint32"] == has32 and st["uinteger"] == u32


def test_permutation_golden():
    z = np.load(GOLDEN / "rng.npz")
    for case, want in zip(z["perm_cases"], z["perm_out"]):
        sd, n = int(case[0]), int(case[1])
        got, _ = oracle.permutation(oracle.pcg64_state(sd), n)
        assert got.tolist() == want[:n].tolist()


@pytest.mark.parametrize("d", [1, 2, 7, 16, 32, 96, 128, 200, 960])
def test_squared_l2_golden(d):
    z = np.load(GOLDEN / "l2.npz")
    got = oracle.squared_l2(z[f"x{d}"], z[f"q{d}"])
    assert np.array_equal(got, z[f"sq{d}"])


def test_keep_count_and_cooldown_goldens():
    # direction.py goldens (reference tests/test_direction.py)
    assert oracle.keep_count(32, 0.5) == 16
    assert oracle.keep_count(8, 0.5) == 4
    assert oracle.keep_count(3, 0.5) == 2  # half-up rounding
    assert oracle.keep_count(1, 0.99) == 1
    assert oracle.in_cooldown(14, 20, 0.3)
    assert not oracle.in_cooldown(13, 20, 0.3)
    assert oracle.in_cooldown(0, 10, 1.0)
    assert not oracle.in_cooldown(9, 10, 0.0)


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c[0])
def test_oracle_runs_match_reference_small(case):
    name, params, mode, prefix = case
    z, _, queries, _, ctxs = load("small")
    got = oracle_dict(oracle.run(queries, ctxs, params, mode))
    assert_run_equal(got, expected(z, prefix), name)


@pytest.mark.parametrize("case", sift_cases(), ids=lambda c: c[0])
def test_oracle_runs_match_reference_sift128(case):
    name, params, mode, prefix = case
    z, _, queries, _, ctxs = load("sift128")
    got = oracle_dict(oracle.run(queries, ctxs, params, mode))
    assert_run_equal(got, expected(z, prefix), name)


def test_oracle_threads_do_not_change_results():
    z, _, queries, _, ctxs = load("small")
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=29, ghost_enabled=True)
    a = oracle_dict(oracle.run(queries, ctxs, params, "pipelined", threads=1))
    b = oracle_dict(oracle.run(queries, ctxs, params, "pipelined", threads=8))
    assert_run_equal(a, b, "threads")


def test_oracle_single_search_cases():
    z = np.load(GOLDEN / "search.npz")

    class Ctx:
        pass

    # complete graph == exact kNN (reference test_search.py:105-115)
    c = Ctx()
    c.vectors = z["complete_vectors"]
    c.adj = z["complete_adj"]
    c.global_ids = np.arange(64, dtype=np.int32)
    c.direction = None
    p = SearchParams(k=10, l=16, m=8, r=2, max_iter=20, seed=5)
    for qi in range(10):
        q = c.vectors[qi] + np.float32(0.01)
        res, _ = oracle.search(q, c, p, seeds=(0,), rng_state=oracle.pcg64_state(prng.derive_seed(5, 4, qi, 0)))
        assert res["ids"].tolist() == z["complete_ids"][qi].tolist()
        assert np.array_equal(res["dists"], z["complete_dists"][qi])
    # buffer-cap visit order (test_search.py:197-205)
    c = Ctx()
    c.vectors = np.arange(10, dtype=np.float32)[:, None]
    c.adj = z["line_adj"]
    c.global_ids = np.arange(10, dtype=np.int32)
    c.direction = None
    p = SearchParams(k=1, l=4, m=1, r=1, max_iter=2, seed=0, buffer_cap=5, log_visits=True)
    res, _ = oracle.search(np.zeros(1, np.float32), c, p, seeds=(9,),
                           rng_state=oracle.pcg64_state(prng.derive_seed(0, 4, 0, 0)))
    assert res["visited_ids"].tolist() == z["line_visited"].tolist()
    assert res["counters"]["total_visits"] == int(z["line_total_visits"])
    # visit log + rng round trip
    c = Ctx()
    c.vectors = z["visit_vectors"]
    c.adj = z["visit_adj"]
    c.global_ids = np.arange(c.vectors.shape[0], dtype=np.int32)
    c.direction = None
    p = SearchParams(k=5, l=16, m=16, r=4, max_iter=12, seed=2, log_visits=True)
    res, st = oracle.search(c.vectors[3], c, p, rng_state=oracle.pcg64_state(prng.derive_seed(2, 4, 3, 0)))
    assert res["visited_ids"].tolist() == z["visit_log"].tolist()
    assert res["ids"].tolist() == z["visit_ids"].tolist()
    cn = res["counters"]
    assert [cn[k] for k in ("iterations", "distance_computations", "total_visits", "nodes_expanded",
                            "dgs_skipped", "inserted_total")] == z["visit_counters"].tolist()
    after = z["visit_rng_after"]
    assert st["state"]["state"] == (int(after[0]) << 64) | int(after[1])
    assert st["has_uint32"] == int(after[2]) and st["uinteger"] == int(after[3])
