"""GPU runner CLI (paper_2507_17094_b200.cli): the
reference's search / bench / eval subcommands (shardann/cli.py:236-316) on
the B200 path.  CPU tests cover config resolution, the vecs files and eval;
the GPU tests run `search` and `bench` on the golden 4-shard fixture and
compare with what the reference itself produced."""

import json

import numpy as np
import pytest

from paper_2507_17094_b200 import cli


def test_config_file_rules(tmp_path):
    conf = tmp_path / "c.conf"
    conf.write_text("# comment\nmax-iter = 12   # trailing\nghost = true\ndiscard = 0.5\nselection = direction\n"
                    "degree = 32\n")
    args = cli.parser().parse_args(["search", "--data", "a", "--queries", "b", "--index", "c", "--metrics", "d",
                                    "--out-ids", "e", "--out-dists", "f", "--config", str(conf), "--l", "48"])
    cfg = cli.resolve(args)
    assert cfg["max_iter"] == 12 and cfg["ghost"] is True and cfg["discard"] == 0.5
    assert cfg["selection"] == "direction" and cfg["l"] == 48 and cfg["k"] == 10  # flag > file > default
    args2 = cli.parser().parse_args(["search", "--data", "a", "--queries", "b", "--index", "c", "--metrics", "d",
                                     "--out-ids", "e", "--out-dists", "f", "--config", str(conf), "--no-ghost"])
    assert cli.resolve(args2)["ghost"] is False
    conf.write_text("bogus = 1\n")
    with pytest.raises(cli.CliError, match="unknown config keys"):
        cli.resolve(args)
    conf.write_text("l 64\n")
    with pytest.raises(cli.CliError, match="expected 'key = value'"):
        cli.resolve(args)


def test_vecs_round_trip_and_errors(tmp_path):
    f = np.random.default_rng(0).standard_normal((7, 5)).astype(np.float32)
    i = np.arange(21, dtype=np.int32).reshape(7, 3)
    cli._write_vecs(tmp_path / "x.fvecs", f)
    cli._write_vecs(tmp_path / "x.ivecs", i)
    assert np.array_equal(cli._vecs(tmp_path / "x.fvecs", "f"), f)
    assert np.array_equal(cli._vecs(tmp_path / "x.ivecs", "i"), i)
    (tmp_path / "bad.fvecs").write_bytes(np.array([3, 1, 2], np.int32).tobytes())
    with pytest.raises(cli.CliError, match="not a fvecs file"):
        cli._vecs(tmp_path / "bad.fvecs", "f")


def test_eval_recall(tmp_path, capsys):
    truth = np.array([[1, 2, 3], [4, 5, 6]], np.int32)
    got = np.array([[3, 2, 9], [7, 8, 9]], np.int32)
    cli._write_vecs(tmp_path / "t.ivecs", truth)
    cli._write_vecs(tmp_path / "r.ivecs", got)
    rc = cli.main(["eval", "--results", str(tmp_path / "r.ivecs"), "--truth-ids", str(tmp_path / "t.ivecs"),
                   "--k", "3", "--out", str(tmp_path / "e.json")])
    assert rc == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep == {"k": 3, "queries": 2, "recall_at_k": pytest.approx((2 / 3 + 0) / 2)}
    assert json.loads((tmp_path / "e.json.manifest.json").read_text())["command"] == "eval"
    assert cli.main(["eval", "--results", str(tmp_path / "missing.ivecs"), "--truth-ids",
                     str(tmp_path / "t.ivecs")]) == 1


def _fixture_files(tmp_path):
    from golden_util import load

    from paper_2507_17094_b200.container import serialize_index

    z, base, queries, index, ctxs = load("small")
    cli._write_vecs(tmp_path / "base.fvecs", base.data)
    cli._write_vecs(tmp_path / "q.fvecs", queries)
    serialize_index(index, tmp_path / "idx.pwix")
    return z


@pytest.mark.gpu
def test_search_command_matches_reference(tmp_path):
    """`search --mode pipelined` with the golden arm's parameters writes the
    reference's final ids and distances, and a metrics document."""
    from golden_util import expected

    z = _fixture_files(tmp_path)
    args = ["search", "--data", str(tmp_path / "base.fvecs"), "--queries", str(tmp_path / "q.fvecs"),
            "--index", str(tmp_path / "idx.pwix"), "--out-ids", str(tmp_path / "r.ivecs"),
            "--out-dists", str(tmp_path / "r.fvecs"), "--metrics", str(tmp_path / "m.json"),
            "--mode", "pipelined", "--k", "10", "--l", "32", "--m", "32", "--r", "4", "--max-iter", "24",
            "--seed", "17", "--selection", "direction", "--discard", "0.5", "--cooldown", "0.3", "--ghost",
            "--ghost-max-iter", "6"]
    assert cli.main(args) == 0
    want = expected(z, "arm06_pipelined_")
    assert np.array_equal(cli._vecs(tmp_path / "r.ivecs", "i"), want["final_ids"])
    assert np.array_equal(cli._vecs(tmp_path / "r.fvecs", "f"), want["final_dists"])
    doc = json.loads((tmp_path / "m.json").read_text())
    assert doc["mode"] == "pipelined" and doc["num_queries"] == want["final_ids"].shape[0]
    man = json.loads((tmp_path / "r.ivecs.manifest.json").read_text())
    assert man["command"] == "search" and len(man["index_checksum"]) > 0


@pytest.mark.gpu
def test_bench_command_sweep(tmp_path):
    """`bench` writes one CSV row per budget with recall growing with it."""
    from paper_2507_17094_b200.metrics import read_sweep_csv

    z = _fixture_files(tmp_path)
    truth = np.asarray(z["truth_ids"] if "truth_ids" in z.files else z["final_ids"]
                       if "final_ids" in z.files else None)
    if truth is None or truth.ndim != 2:
        from paper_2507_17094_b200 import exact

        truth, _ = exact.exact_knn_batch(z["base"], z["queries"], 10)
    cli._write_vecs(tmp_path / "t.ivecs", np.asarray(truth, np.int32))
    rc = cli.main(["bench", "--data", str(tmp_path / "base.fvecs"), "--queries", str(tmp_path / "q.fvecs"),
                   "--index", str(tmp_path / "idx.pwix"), "--truth-ids", str(tmp_path / "t.ivecs"),
                   "--budgets", "2,8,24", "--seeds", "0,1", "--out", str(tmp_path / "s.csv"), "--l", "32",
                   "--mode", "pipelined"])
    assert rc == 0
    rows = read_sweep_csv(tmp_path / "s.csv")
    assert [r["budget"] for r in rows] == [2, 8, 24]
    assert rows[0]["recall"] <= rows[-1]["recall"] and rows[-1]["recall"] > 0.5
