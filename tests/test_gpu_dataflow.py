"""Dataflow ring (pw_search_dataflow): the pipelined path extension as one
persistent K1 per shard, entries handed over through inboxes with release /
acquire stores instead of stage barriers.  On one GPU the N shards run
concurrently (N streams, SMs/N CTAs each) -- the same protocol the
one-GPU-per-shard ring runs over NVLink peer mappings.  Results must equal
the reference pipelined run (oracle) bit for bit, in any interleaving."""

import numpy as np
import pytest
import torch

import oracle
from df_util import assert_same, run_dict, tensor_shard
from golden_util import load, oracle_dict
from index_util import clustered, make_contexts
from paper_2507_17094_b200 import device as dv
from paper_2507_17094_b200.search import SearchParams

pytestmark = pytest.mark.gpu

ARMS = [
    dict(k=10, l=64, m=64, r=8, max_iter=64, seed=1),
    dict(k=10, l=128, m=64, r=8, max_iter=64, seed=2, selection="direction", discard_ratio=0.5,
         cooldown_ratio=0.3, ghost_enabled=True, ghost_max_iter=8),
    dict(k=10, l=96, m=64, r=4, max_iter=10, seed=3, selection="random", discard_ratio=0.5,
         seed_mode="mixed", ghost_enabled=True),
]


@pytest.fixture(scope="module")
def rings():
    out = {}
    for n_shards in (2, 3, 4):
        x = clustered(16000 + 400, 96, 256, 0.08, seed=40 + n_shards)
        ctxs = make_contexts(x[:16000], n_shards, 32, seed=n_shards)
        out[n_shards] = (np.ascontiguousarray(x[16000:]), ctxs, [tensor_shard(c) for c in ctxs])
    return out


def _run(queries, shards, params, tuning=None, reps=1):
    q = queries.shape[0]
    tq = torch.from_numpy(queries).cuda()
    run = dv.DeviceRun(q, len(shards), params.k, "cuda")
    df = dv.LocalDataflow(shards, q, params.k, "cuda")
    for _ in range(reps):  # later runs reuse the inboxes (epoch-tagged, never reset)
        run.shard_ids.fill_(7)
        run.s64.fill_(-5)
        df.run(params, tq, run, tuning=tuning)
    torch.cuda.synchronize()
    for sh in shards:
        dv.check_shard(sh)
    return run_dict(run.shard_ids.cpu().numpy(), run.shard_dists.cpu().numpy(),
                    run.final_ids.cpu().numpy(), run.final_dists.cpu().numpy(),
                    run.s32.cpu().numpy(), run.s64.cpu().numpy())


@pytest.mark.parametrize("n_shards", [2, 3, 4])
@pytest.mark.parametrize("arm", range(len(ARMS)))
def test_local_dataflow_matches_oracle(rings, n_shards, arm):
    queries, ctxs, shards = rings[n_shards]
    params = SearchParams(**ARMS[arm])
    want = oracle_dict(oracle.run(queries, ctxs, params, "pipelined"))
    got = _run(queries, shards, params, reps=2)
    assert_same(got, want, f"dataflow N={n_shards} arm={arm}")
    lossy = _run(queries, shards, params, tuning={"flags": 2})
    assert_same(lossy, want, f"dataflow lossy N={n_shards} arm={arm}", lossy=True)


def test_local_dataflow_golden_fixture():
    """The reference's own 4-shard pipelined output (tests/golden/small.npz)."""
    from golden_util import expected

    z, base, queries, index, ctxs = load("small")
    params = SearchParams(k=10, l=32, m=32, r=4, max_iter=24, seed=17, selection="direction",
                          discard_ratio=0.5, cooldown_ratio=0.3, ghost_enabled=True, ghost_max_iter=6)
    got = _run(np.ascontiguousarray(queries, np.float32), [tensor_shard(c) for c in ctxs], params)
    want = expected(z, "arm06_pipelined_")
    assert_same(got, want, "golden arm06 dataflow")


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_dataflow_ring(tmp_path, world):
    """One process per shard exchanging entries through CUDA IPC peer
    mappings (ring.DataflowRing) -- here the ranks share the one GPU, on an
    8-GPU box each owns one and the stores cross NVLink."""
    import json
    import socket
    import subprocess
    import sys
    from pathlib import Path

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "df.json"
    worker = Path(__file__).resolve().parent / "df_ring_worker.py"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
                        "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(worker), str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    report = json.loads(out.read_text())
    assert report and all(v == "ok" for v in report.values()), report


# Opt-in path-extension knobs (not the reference's behaviour): top-F entries
# forwarded per query and smaller budgets for stages >= 1.  The oracle runs
# the same knobs (oracle.run(..., ext=...)), so the GPU paths must still agree
# with it bit for bit -- through the stage schedule, the dataflow ring and pw_run.
EXT = [dict(forward_count=2), dict(forward_count=4, late_l=64), dict(late_l=48, late_max_iter=6),
       dict(forward_count=3, late_max_iter=8)]


@pytest.mark.parametrize("n_shards", [2, 4])
@pytest.mark.parametrize("arm", [0, 1, 2])
@pytest.mark.parametrize("ext", range(len(EXT)))
def test_extension_knobs_match_oracle(rings, n_shards, arm, ext):
    queries, ctxs, shards = rings[n_shards]
    params = SearchParams(**ARMS[arm])
    knobs = EXT[ext]
    want = oracle_dict(oracle.run(queries, ctxs, params, "pipelined", ext=knobs))
    got = _run(queries, shards, params, tuning=dict(knobs), reps=2)
    assert_same(got, want, f"dataflow ext={knobs} N={n_shards} arm={arm}")
    # stage-synchronous schedule (N x N pw_search_stage launches)
    q = queries.shape[0]
    run = dv.DeviceRun(q, len(shards), params.k, "cuda")
    dv.run_local(shards, params, torch.from_numpy(queries).cuda(), "pipelined", run, tuning=dict(knobs))
    torch.cuda.synchronize()
    got2 = run_dict(run.shard_ids.cpu().numpy(), run.shard_dists.cpu().numpy(), run.final_ids.cpu().numpy(),
                    run.final_dists.cpu().numpy(), run.s32.cpu().numpy(), run.s64.cpu().numpy())
    assert_same(got2, want, f"stages ext={knobs} N={n_shards} arm={arm}")
    # the host API (pw_run, pinned host buffers) with the same knobs
    import paper_2507_17094_b200 as pw
    from golden_util import result_dict

    got3 = result_dict(pw.run_pipelined(pw.Dataset(queries), None, None, params, contexts=ctxs,
                                        tuning=dict(knobs)))
    for key in ("final_ids", "final_dists", "shard_ids", "shard_dists"):
        assert np.array_equal(got3[key], want[key]), (knobs, key)
    assert np.array_equal(got3["comm"], want["comm"])


def test_extension_knob_validation(rings):
    queries, ctxs, shards = rings[2]
    params = SearchParams(**ARMS[0])
    q = torch.from_numpy(queries).cuda()
    run = dv.DeviceRun(q.shape[0], 2, params.k, "cuda")
    with pytest.raises(ValueError, match="forward_count"):
        dv.run_local(shards, params, q, "pipelined", run, tuning={"forward_count": 11})
    with pytest.raises(ValueError, match="k <= l"):
        dv.run_local(shards, params, q, "pipelined", run, tuning={"late_l": 5})
