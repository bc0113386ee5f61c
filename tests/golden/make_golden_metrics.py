"""Golden fixtures for run instrumentation (shardann/metrics.py
and the recall helpers of shardann/oracle.py), made by the reference itself.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden_metrics.py

Writes tests/golden/metrics.json: for the conftest small fixture (4 shards,
d=16) and two arms of small.npz (arm 3 = full selection + ghost + mixed
seeding; arm 5 = direction 0.5 + neighbors seeding), per mode:
* collect_metrics(result) (both classification modes) and the JSON document
  write_metrics_json writes (wall time / config fixed),
* cost_model_report(params, d, degree, result),
* mean_recall against exact_knn_batch at k,
* sweep(...) rows for budgets (2, 6, 24) with seeds (17, 18).
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import sys
import tempfile
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import shardann as sa  # noqa: E402
from shardann import metrics as M  # noqa: E402

OUT = Path(__file__).resolve().parent
SMALL_BASE = dict(k=10, l=32, m=32, r=4, max_iter=24, seed=17, cooldown_ratio=0.3, ghost_max_iter=6)
ARMS = {3: dict(selection="full", discard_ratio=0.0, ghost_enabled=True, seed_mode="mixed"),
        5: dict(selection="direction", discard_ratio=0.5, ghost_enabled=False, seed_mode="mixed")}
BUDGETS = (2, 6, 24)
SEEDS = (17, 18)


def main():
    full = sa.gen_synthetic(4100, 16, 32, 0.2, seed=99)
    base = sa.Dataset(full.data[:4000])
    queries = sa.Dataset(full.data[4000:])
    index, _ = sa.build_index(base, 4, 16, seed=5, rho=0.05, ghost_degree=8)
    truth = sa.exact_knn_batch(base, queries, 10)
    contexts = sa.build_contexts(index, base)
    out = {"budgets": BUDGETS, "seeds": SEEDS, "arms": {}}
    for arm, kw in ARMS.items():
        params = sa.SearchParams(**SMALL_BASE, **kw)
        per_mode = {}
        for mode, runner in (("baseline", sa.run_sharded_baseline), ("pipelined", sa.run_pipelined)):
            res = runner(queries, index, base, params, contexts=contexts)
            m_q = M.collect_metrics(res)
            m_t = M.collect_metrics(res, mode="topk")
            recall = sa.mean_recall(truth, res.neighbor_lists(), params.k)
            cost = M.cost_model_report(params, base.d, 16, res)
            with tempfile.TemporaryDirectory() as td:
                doc = M.write_metrics_json(Path(td) / "m.json", res, params, cost_model=cost, recall=recall,
                                           wall_time_s=1.5, config={"arm": arm})
                text = (Path(td) / "m.json").read_text()
            rows = M.sweep(queries, index, base, truth, params, BUDGETS, mode=mode, seeds=SEEDS,
                           contexts=contexts)
            with tempfile.TemporaryDirectory() as td:
                M.write_sweep_csv(rows, Path(td) / "s.csv")
                csv_text = (Path(td) / "s.csv").read_text()
            per_mode[mode] = {
                "classify_queue": list(M.classify_visits(res)),
                "classify_topk": list(M.classify_visits(res, "topk")),
                "metrics_queue": {**m_q.totals_dict(), "per_stage": m_q.per_stage},
                "metrics_topk": m_t.totals_dict(),
                "recall": recall,
                "cost_model": cost,
                "metrics_json": doc,
                "metrics_json_text": text,
                "sweep": rows,
                "sweep_csv": csv_text,
            }
        out["arms"][str(arm)] = {"params": {**SMALL_BASE, **kw}, "modes": per_mode}
    # the sweep's replace(params, max_iter=budget, seed=seed) is a plain field copy
    assert replace(sa.SearchParams(**SMALL_BASE), max_iter=2).max_iter == 2
    (OUT / "metrics.json").write_text(json.dumps(out, indent=1, sort_keys=True, default=_ser) + "\n")


def _ser(o):
    if hasattr(o, "item"):
        return o.item()
    if isinstance(o, tuple):
        return list(o)
    raise TypeError(type(o))


if __name__ == "__main__":
    main()
