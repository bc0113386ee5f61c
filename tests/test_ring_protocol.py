"""Model check of ring.DataflowRing's device-side batch protocol (CPU).

Every rank's CUDA stream is modelled as a FIFO of the operations
DataflowRing.submit enqueues (reset / signal / wait / K1 / K2), and one
persistent K1 as a process that needs the entries of its stage-s > 0 tasks
from the previous rank's K1 of the SAME batch.  A random scheduler advances
any stream whose head can make progress.  The properties the protocol must
give, for every N, depth and interleaving:

* no deadlock: all batches complete;
* a slot's inbox is never overwritten by batch e + depth before the
  consumer finished batch e (else a stage-s task would wait for an epoch
  that was overwritten);
* rank 0's result slot is never reset, or written by batch e + depth, before
  the K2 of batch e ran;
* K2 of batch e runs only after every rank's K1 of batch e finished.
"""

import random

import pytest


def simulate(N: int, depth: int, batches: int, seed: int) -> None:
    rnd = random.Random(seed)
    landed = [[0] * depth for _ in range(N)]  # rank 0's words, one per (rank, slot)
    done = [0] * depth
    inbox_epoch = [[0] * depth for _ in range(N)]  # epoch written into rank g's inbox slot
    consumed = [[0] * depth for _ in range(N)]     # last epoch whose inbox slot rank g fully read
    k1_done = [[False] * (batches + 1) for _ in range(N)]
    k1_started = [[False] * (batches + 1) for _ in range(N)]
    reduced = [0] * depth      # last epoch reduced (K2) per slot
    streams = []
    for g in range(N):
        ops = []
        for e in range(1, batches + 1):
            b = e % depth
            if e > depth:
                if g == 0:
                    ops += [("reset", e, b), ("signal_done", e - depth, b)]
                else:
                    ops.append(("wait_done", e - depth, b))
            ops += [("k1", e, b), ("signal_landed", e, b)]
            if g == 0:
                ops += [("wait_landed", e, b), ("k2", e, b)]
        streams.append(ops)

    def can_run(g, op):
        kind, e, b = op
        if kind == "wait_done":
            return done[b] >= e
        if kind == "wait_landed":
            return all(landed[r][b] >= e for r in range(N))
        if kind == "k1":
            # the persistent kernel may start; it finishes when the previous
            # rank's K1 of the same batch has produced its entries (stage s > 0)
            return True
        return True

    pos = [0] * N
    running = [None] * N  # (e, b) of a started K1 waiting for entries
    steps = 0
    while any(pos[g] < len(streams[g]) for g in range(N)):
        steps += 1
        assert steps < 100_000, "livelock"
        ready = []
        for g in range(N):
            if running[g] is not None:
                e, b = running[g]
                prev = (g - 1) % N
                if N == 1 or k1_started[prev][e]:
                    ready.append(g)
                continue
            if pos[g] < len(streams[g]) and can_run(g, streams[g][pos[g]]):
                ready.append(g)
        assert ready, f"deadlock at {pos} running={running}"
        g = rnd.choice(ready)
        if running[g] is not None:
            e, b = running[g]
            # K1 finishes: every stage-s > 0 entry it read was epoch e
            assert N == 1 or inbox_epoch[g][b] == e, "entry of another batch"
            consumed[g][b] = e
            k1_done[g][e] = True
            running[g] = None
            pos[g] += 1
            continue
        kind, e, b = streams[g][pos[g]]
        if kind == "k1":
            # a running K1 stores into the next rank's inbox slot b and into
            # rank 0's result slot b
            nxt = (g + 1) % N
            assert consumed[nxt][b] >= e - depth, "inbox slot overwritten before it was consumed"
            inbox_epoch[nxt][b] = e
            assert reduced[b] >= e - depth, "result slot written before its previous batch was reduced"
            k1_started[g][e] = True
            running[g] = (e, b)
            continue
        if kind == "reset":
            assert reduced[b] == e - depth, "slot reset before its K2"
        elif kind == "signal_done":
            done[b] = e
        elif kind == "signal_landed":
            landed[g][b] = e
        elif kind == "k2":
            assert all(k1_done[r][e] for r in range(N)), "K2 before every K1 of its batch"
            reduced[b] = e
        pos[g] += 1
    assert all(all(k1_done[g][1:]) for g in range(N))


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_dataflow_batch_protocol(N, depth):
    for seed in range(25):
        simulate(N, depth, batches=7, seed=seed)
