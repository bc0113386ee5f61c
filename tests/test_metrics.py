"""Run instrumentation against the reference's own outputs
(tests/golden/metrics.json, made by make_golden_metrics.py), mirroring the
reference's tests/test_metrics.py (visit identity :34-41, unknown mode
:44-46, cost model :59-98, sweep + CSV :101-141, JSON schema :144-).

CPU tests fold the reference-produced PipelineResults of small.npz through
this package's metrics; GPU tests produce the results (and the sweeps) with
the CUDA path and must give the same documents.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import golden_util as gu
from paper_2507_17094_b200 import metrics as M
from paper_2507_17094_b200.pipeline import NeighborList, PipelineResult, StageStats
from paper_2507_17094_b200.search import SearchParams

GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "metrics.json").read_text())
CASES = [(arm, mode) for arm in sorted(G["arms"]) for mode in ("baseline", "pipelined")]


def _json_norm(x):
    return json.loads(json.dumps(x, sort_keys=True))


def _golden_result(z, arm: int, mode: str, k: int) -> PipelineResult:
    want = gu.expected(z, f"arm{arm:02d}_{mode}_")
    n = want["shard_ids"].shape[1]
    stages = [StageStats(**{f: want[f][s] for f in gu.STAT_FIELDS}) for s in range(n)]
    return PipelineResult(mode=mode, k=k, shard_ids=want["shard_ids"], shard_dists=want["shard_dists"],
                          final_ids=want["final_ids"], final_dists=want["final_dists"], stages=stages,
                          comm_stage_bytes=want["comm"])


@pytest.fixture(scope="module")
def small():
    return gu.load("small")


def _truth(z):
    return [NeighborList(i, z["truth_ids"][i], z["truth_dists"][i]) for i in range(z["truth_ids"].shape[0])]


def _check_docs(res, params, g, tmp_path, d):
    assert list(M.classify_visits(res)) == g["classify_queue"]
    assert list(M.classify_visits(res, "topk")) == g["classify_topk"]
    mq = M.collect_metrics(res)
    assert _json_norm({**mq.totals_dict(), "per_stage": mq.per_stage}) == g["metrics_queue"]
    assert _json_norm(M.collect_metrics(res, mode="topk").totals_dict()) == g["metrics_topk"]
    tot = mq.totals_dict()
    assert tot["total_visits"] == tot["discarded_visits"] + tot["retained_visits"]  # visit identity
    cost = M.cost_model_report(params, d, 16, res)
    assert _json_norm(cost) == g["cost_model"]
    path = tmp_path / "m.json"
    doc = M.write_metrics_json(path, res, params, cost_model=cost, recall=g["recall"], wall_time_s=1.5,
                               config={"arm": int(g["metrics_json"]["config"]["arm"])})
    assert _json_norm(doc) == g["metrics_json"]
    assert path.read_text() == g["metrics_json_text"]


@pytest.mark.parametrize("arm,mode", CASES)
def test_metrics_of_reference_results(arm, mode, small, tmp_path):
    z = small[0]
    g = G["arms"][arm]["modes"][mode]
    params = SearchParams(**G["arms"][arm]["params"])
    res = _golden_result(z, int(arm), mode, params.k)
    assert M.mean_recall(_truth(z), res.neighbor_lists(), params.k) == pytest.approx(g["recall"], abs=0)
    _check_docs(res, params, g, tmp_path, z["base"].shape[1])


def test_classify_rejects_unknown_mode(small):
    res = _golden_result(small[0], 3, "baseline", 10)
    with pytest.raises(ValueError, match="unknown classification mode"):
        M.classify_visits(res, "bogus")


def test_cost_model_detects_mismatch(small):
    res = _golden_result(small[0], 3, "pipelined", 10)
    res.comm_stage_bytes = res.comm_stage_bytes.copy()
    res.comm_stage_bytes[0, 0] += 4
    with pytest.raises(RuntimeError, match="communication accounting mismatch"):
        M.cost_model_report(SearchParams(**G["arms"]["3"]["params"]), 16, 16, res)


def test_sweep_csv_round_trip_matches_reference(tmp_path):
    for arm, mode in CASES:
        g = G["arms"][arm]["modes"][mode]
        path = tmp_path / f"{arm}{mode}.csv"
        M.write_sweep_csv(g["sweep"], path)
        assert path.read_text() == g["sweep_csv"]
        assert M.read_sweep_csv(path) == g["sweep"]


def test_recall_errors():
    a = NeighborList(0, np.arange(3, dtype=np.int32), np.zeros(3, np.float32))
    with pytest.raises(ValueError, match="at least k=5"):
        M.recall_at_k(a, a, 5)
    with pytest.raises(ValueError, match="length mismatch"):
        M.mean_recall([a], [a, a], 3)
    with pytest.raises(ValueError, match="requires ground truth"):
        M.sweep(None, None, None, None, SearchParams(k=1, l=2, m=2, r=1, max_iter=1), [1])


# ------------------------------------------------------------------ GPU tests


@pytest.mark.gpu
@pytest.mark.parametrize("arm,mode", CASES)
def test_gpu_metrics_and_sweep_match_reference(arm, mode, small, tmp_path):
    from paper_2507_17094_b200.pipeline import run_pipelined, run_sharded_baseline

    z, base, queries, index, ctxs = small
    from paper_2507_17094_b200.data import Dataset

    qds = Dataset(queries)
    g = G["arms"][arm]["modes"][mode]
    params = SearchParams(**G["arms"][arm]["params"])
    runner = run_pipelined if mode == "pipelined" else run_sharded_baseline
    res = runner(qds, index, base, params, contexts=ctxs)
    assert M.mean_recall(_truth(z), res.neighbor_lists(), params.k) == g["recall"]
    _check_docs(res, params, g, tmp_path, base.d)
    rows = M.sweep(qds, index, base, _truth(z), params, G["budgets"], mode=mode, seeds=G["seeds"],
                   contexts=ctxs)
    assert rows == g["sweep"]


@pytest.mark.gpu
def test_gpu_exact_knn_lists_match_reference_truth(small):
    z, base, queries, _, _ = small
    got = M.exact_knn_batch(base, queries, 10)
    for i, nl in enumerate(got):
        assert np.array_equal(nl.ids, z["truth_ids"][i])
        assert np.array_equal(nl.dists, z["truth_dists"][i])
