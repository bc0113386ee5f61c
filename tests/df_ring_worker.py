"""torchrun worker for test_gpu_dataflow.py::test_multiprocess_dataflow_ring:
one process per shard (ranks may share a GPU), ring.DataflowRing over CUDA
IPC peer mappings, rank 0 checks the result against the CPU oracle.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/df_ring_worker.py OUT.json
"""
import json
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(rank % ndev)
    dist.init_process_group("gloo")
    import oracle
    from df_util import assert_same, run_dict, tensor_shard
    from golden_util import oracle_dict
    from index_util import clustered, make_contexts
    from paper_2507_17094_b200 import ring
    from paper_2507_17094_b200.search import SearchParams

    x = clustered(12000 + 300, 96, 256, 0.08, seed=77)
    ctxs = make_contexts(x[:12000], world, 32, seed=world)
    queries = np.ascontiguousarray(x[12000:])
    shard = tensor_shard(ctxs[rank])
    sms = torch.cuda.get_device_properties(rank % ndev).multi_processor_count
    per_gpu = -(-world // ndev)  # ranks sharing one GPU split its SMs
    eng = ring.DataflowRing(shard, queries.shape[0], 10, rank, world, torch.device("cuda", rank % ndev),
                            sm_limit=sms // per_gpu if per_gpu > 1 else 0)
    tq = torch.from_numpy(queries).cuda()
    report = {}
    for name, kw, mode in (
            ("pipelined_ghost_dgs", dict(selection="direction", discard_ratio=0.5, cooldown_ratio=0.3,
                                         ghost_enabled=True, ghost_max_iter=8), "pipelined"),
            ("pipelined_full", dict(), "pipelined"),
            ("baseline", dict(), "baseline")):
        params = SearchParams(k=10, l=96, m=64, r=8, max_iter=64, seed=5, **kw)
        for _ in range(2):  # second run reuses the inboxes (new epoch)
            eng.run(tq, params, mode)
        want = oracle_dict(oracle.run(queries, ctxs, params, mode)) if rank == 0 else None

        def check(tag):
            slot = eng.last % eng.depth
            ids, dists, s32, s64 = (a.t.cpu().numpy() for a in eng.res[slot])
            got = run_dict(ids, dists, eng.final_ids[slot].cpu().numpy(), eng.final_dists[slot].cpu().numpy(),
                           s32, s64)
            try:
                assert_same(got, want, tag)
                report[tag] = "ok"
            except AssertionError as e:
                report[tag] = str(e)

        if rank == 0:
            check(name)
        # a stream of batches with no host synchronisation in between: slots
        # and inboxes are reused under the device-side landed/done protocol
        for _ in range(5):
            eng.submit(tq, params, mode)
        eng.sync()
        if rank == 0:
            check(name + "_pipelined_batches")
    dist.barrier()
    if rank == 0:
        Path(out_path).write_text(json.dumps(report))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
