"""GPU runner CLI for the search path: the reference's
`search`, `bench` and `eval` subcommands (shardann/cli.py:236-316) with the
same flags, config-file rules and output files, running on the B200 through
this package's runners.  Index building, data generation and ground truth
stay with shardann's own CLI (`build`, `gen`, `truth`); their files (.pwix,
fvecs, ivecs) are read here unchanged.

    python -m paper_2507_17094_b200.cli search --data base.fvecs --queries q.fvecs \\
        --index idx.pwix --out-ids r.ivecs --out-dists r.fvecs --metrics m.json --mode pipelined
    python -m paper_2507_17094_b200.cli bench --data ... --index ... --truth-ids t.ivecs \\
        --budgets 8,16,32 --seeds 0,1 --out sweep.csv
    python -m paper_2507_17094_b200.cli eval --results r.ivecs --truth-ids t.ivecs --k 10

Precedence is flag > `--config` file (`key = value` lines, `#` comments,
dashes or underscores) > built-in default, as in the reference; every run
writes `<primary output>.manifest.json` (resolved config, seed, outputs,
index checksum).  Errors are one line on stderr and exit code 1.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

# shardann/cli.py DEFAULTS restricted to the keys these subcommands read
SEARCH_KEYS = ("k", "l", "m", "r", "max_iter", "seed", "selection", "discard", "cooldown", "ghost",
               "ghost_max_iter", "seed_mode", "threads", "mode")
DEFAULTS = dict(k=10, l=64, m=64, r=8, max_iter=64, seed=0, selection="full", discard=0.0, cooldown=0.3,
                ghost=False, ghost_max_iter=8, seed_mode="neighbors", threads=1, mode="baseline")
# keys shardann's config files may hold for its other subcommands: accepted, unused here
OTHER_KEYS = {"degree", "shards", "rho", "ghost_degree", "n", "d", "clusters", "spread", "queries"}


class CliError(Exception):
    """One line on stderr, exit code 1."""


# ------------------------------------------------------------------ files
def _vecs(path: Path, kind: str) -> np.ndarray:
    """(rows, dim) array of an fvecs (kind 'f') / ivecs (kind 'i') file: each
    row is an int32 dimension followed by that many 4-byte values."""
    raw = np.fromfile(path, dtype=np.int32)
    if raw.size == 0:
        return np.zeros((0, 0), np.float32 if kind == "f" else np.int32)
    dim = int(raw[0])
    if dim <= 0 or raw.size % (dim + 1):
        raise CliError(f"{path}: not a {kind}vecs file (dimension {dim}, {raw.size * 4} bytes)")
    rows = raw.reshape(-1, dim + 1)
    if np.any(rows[:, 0] != dim):
        raise CliError(f"{path}: rows of different dimensions")
    body = np.ascontiguousarray(rows[:, 1:])
    return body.view(np.float32) if kind == "f" else body


def _write_vecs(path: Path, values: np.ndarray) -> None:
    values = np.ascontiguousarray(values)
    out = np.empty((values.shape[0], values.shape[1] + 1), np.int32)
    out[:, 0] = values.shape[1]
    out[:, 1:] = values.view(np.int32)
    out.tofile(path)


def _path(p) -> Path:
    """Relative paths honour $SHARDANN_DATA_DIR, as the reference's CLI does."""
    p = Path(p)
    root = os.environ.get("SHARDANN_DATA_DIR")
    return Path(root) / p if root and not p.is_absolute() else p


def _existing(p, what: str) -> Path:
    q = _path(p)
    if not q.is_file():
        raise CliError(f"{what} file not found: {q}")
    return q


# ----------------------------------------------------------------- config
def read_config(path) -> dict:
    """`key = value` per line; booleans, ints and floats parsed, else str."""
    out = {}
    for n, line in enumerate(Path(path).read_text().splitlines(), 1):
        body = line.split("#", 1)[0].strip()
        if not body:
            continue
        key, sep, value = body.partition("=")
        if not sep:
            raise CliError(f"{path}:{n}: expected 'key = value', got {line!r}")
        key, value = key.strip().replace("-", "_"), value.strip()
        if value.lower() in ("true", "false"):
            out[key] = value.lower() == "true"
        else:
            for cast in (int, float, str):
                try:
                    out[key] = cast(value)
                    break
                except ValueError:
                    pass
    return out


def resolve(args, keys=SEARCH_KEYS) -> dict:
    conf = read_config(args.config) if getattr(args, "config", None) else {}
    bad = sorted(set(conf) - set(DEFAULTS) - OTHER_KEYS)
    if bad:
        raise CliError(f"unknown config keys: {bad}")
    return {key: next(v for v in (getattr(args, key, None), conf.get(key), DEFAULTS[key]) if v is not None)
            for key in keys}


def search_params(cfg: dict):
    from .search import SearchParams

    try:
        return SearchParams(k=cfg["k"], l=cfg["l"], m=cfg["m"], r=cfg["r"], max_iter=cfg["max_iter"],
                            seed=cfg["seed"], selection=cfg["selection"], discard_ratio=cfg["discard"],
                            cooldown_ratio=cfg["cooldown"], ghost_enabled=cfg["ghost"],
                            ghost_max_iter=cfg["ghost_max_iter"], seed_mode=cfg["seed_mode"])
    except ValueError as e:
        raise CliError(f"invalid search parameters: {e}") from e


def _manifest(primary, command: str, cfg: dict, outputs, checksum: str | None = None) -> None:
    doc = {"command": command, "config": dict(sorted(cfg.items())), "seed": cfg.get("seed"),
           "outputs": [str(o) for o in outputs]}
    if checksum is not None:
        doc["index_checksum"] = checksum
    Path(str(primary) + ".manifest.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def _inputs(args):
    from .container import deserialize_index
    from .data import Dataset

    data = Dataset(_vecs(_existing(args.data, "dataset"), "f"))
    queries = Dataset(_vecs(_existing(args.queries, "query"), "f"))
    index_path = _existing(args.index, "index")
    return data, queries, deserialize_index(index_path), index_path


# ------------------------------------------------------------ subcommands
def cmd_search(args) -> int:
    """shardann/cli.py:236-262 on the GPU runners."""
    from . import pipeline
    from .container import index_file_checksum
    from .metrics import cost_model_report, write_metrics_json

    cfg = resolve(args)
    data, queries, index, index_path = _inputs(args)
    params = search_params(cfg)
    runner = pipeline.run_pipelined if cfg["mode"] == "pipelined" else pipeline.run_sharded_baseline
    print(f"search (B200): mode={cfg['mode']}, {queries.n} queries, {index.n_shards} shards", file=sys.stderr)
    t0 = time.perf_counter()
    res = runner(queries, index, data, params, threads=cfg["threads"])
    wall = time.perf_counter() - t0
    ids_p, dists_p, met_p = _path(args.out_ids), _path(args.out_dists), _path(args.metrics)
    _write_vecs(ids_p, res.final_ids.astype(np.int32))
    _write_vecs(dists_p, res.final_dists.astype(np.float32))
    cost = cost_model_report(params, index.d, index.shards[0].adj.shape[1], res)
    write_metrics_json(met_p, res, params, cost_model=cost, wall_time_s=wall, config=cfg)
    _manifest(ids_p, "search", cfg, [ids_p, dists_p, met_p], index_file_checksum(index_path))
    print(f"search done in {wall:.2f}s", file=sys.stderr)
    return 0


def cmd_bench(args) -> int:
    """shardann/cli.py:289-312: an iteration-budget sweep on the GPU runners."""
    from .container import index_file_checksum
    from .metrics import sweep, write_sweep_csv
    from .pipeline import NeighborList

    cfg = resolve(args)
    data, queries, index, index_path = _inputs(args)
    t_ids = _vecs(_existing(args.truth_ids, "ground-truth"), "i")
    truth = [NeighborList(i, t_ids[i], np.zeros(t_ids.shape[1], np.float32)) for i in range(t_ids.shape[0])]
    try:
        budgets = [int(b) for b in args.budgets.split(",") if b.strip()]
        seeds = [int(s) for s in args.seeds.split(",") if s.strip()]
    except ValueError as e:
        raise CliError(f"budgets/seeds must be comma-separated integers: {e}") from e
    if not budgets:
        raise CliError("no budgets given")
    rows = sweep(queries, index, data, truth, search_params(cfg), budgets, mode=cfg["mode"], seeds=seeds,
                 threads=cfg["threads"])
    out = _path(args.out)
    write_sweep_csv(rows, out)
    _manifest(out, "bench", cfg, [out], index_file_checksum(index_path))
    return 0


def cmd_eval(args) -> int:
    """shardann/cli.py:265-286: recall@k of a results file."""
    cfg = resolve(args, ("k",))
    got = _vecs(_existing(args.results, "results"), "i")
    truth = _vecs(_existing(args.truth_ids, "ground-truth"), "i")
    if truth.shape[0] != got.shape[0]:
        raise CliError(f"results hold {got.shape[0]} queries, truth holds {truth.shape[0]}")
    k = cfg["k"]
    if got.shape[1] < k or truth.shape[1] < k:
        raise CliError(f"need at least k={k} entries per query in results and truth")
    recall = float(np.mean([np.intersect1d(truth[i, :k], got[i, :k]).size / k for i in range(got.shape[0])]))
    report = {"k": k, "queries": int(got.shape[0]), "recall_at_k": recall}
    print(json.dumps(report, sort_keys=True))
    if args.out:
        out = _path(args.out)
        out.write_text(json.dumps(report, indent=2, sort_keys=True) + "\n")
        _manifest(out, "eval", cfg, [out])
    return 0


# ----------------------------------------------------------------- parser
def _search_flags(p) -> None:
    p.add_argument("--k", type=int)
    p.add_argument("--l", type=int)
    p.add_argument("--m", type=int)
    p.add_argument("--r", type=int)
    p.add_argument("--max-iter", dest="max_iter", type=int)
    p.add_argument("--seed", type=int)
    p.add_argument("--selection", choices=["full", "direction", "random"])
    p.add_argument("--discard", type=float)
    p.add_argument("--cooldown", type=float)
    p.add_argument("--ghost", action=argparse.BooleanOptionalAction, default=None)
    p.add_argument("--ghost-max-iter", dest="ghost_max_iter", type=int)
    p.add_argument("--seed-mode", dest="seed_mode", choices=["neighbors", "mixed"])
    p.add_argument("--threads", type=int)
    p.add_argument("--mode", choices=["baseline", "pipelined"])
    p.add_argument("--config")


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2507_17094_b200.cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("search", help="search on the B200; results + metrics")
    for flag in ("--data", "--queries", "--index", "--metrics"):
        p.add_argument(flag, required=True)
    p.add_argument("--out-ids", dest="out_ids", required=True)
    p.add_argument("--out-dists", dest="out_dists", required=True)
    _search_flags(p)
    p.set_defaults(fn=cmd_search)
    p = sub.add_parser("bench", help="iteration-budget sweep on the B200")
    for flag in ("--data", "--queries", "--index", "--budgets", "--out"):
        p.add_argument(flag, required=True)
    p.add_argument("--truth-ids", dest="truth_ids", required=True)
    p.add_argument("--seeds", default="0")
    _search_flags(p)
    p.set_defaults(fn=cmd_bench)
    p = sub.add_parser("eval", help="recall of a results file")
    p.add_argument("--results", required=True)
    p.add_argument("--truth-ids", dest="truth_ids", required=True)
    p.add_argument("--k", type=int)
    p.add_argument("--out")
    p.add_argument("--config")
    p.set_defaults(fn=cmd_eval)
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    try:
        return args.fn(args)
    except (CliError, ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
