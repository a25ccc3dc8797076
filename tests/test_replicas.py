"""The N > 1 path of bench.py on CPU: world_size-2 gloo group, barrier and
the weak-scaling aggregate (sum of units / max of time over ranks)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    from paper_2604_19892_b200.replicas import ReplicaGroup

    g = ReplicaGroup.from_env("gloo")
    g.barrier()
    # rank r did 100 (r + 1) iterations in (r + 2) seconds
    value, units, secs = g.aggregate(100.0 * (rank + 1), float(rank + 2))
    out[rank] = (value, units, secs, g.allmax(rank), g.allsum(1.0))
    g.close()


def test_two_rank_gloo_aggregate():
    ws = 2
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
        res = dict(out)
    for r in range(ws):
        value, units, secs, mx, n = res[r]
        assert units == 300.0 and secs == 3.0
        assert value == pytest.approx(100.0)
        assert mx == 1.0 and n == 2.0


def test_single_rank_is_identity():
    from paper_2604_19892_b200.replicas import ReplicaGroup

    g = ReplicaGroup()
    assert g.aggregate(50.0, 2.0) == (25.0, 50.0, 2.0)
    g.barrier()
    g.close()
