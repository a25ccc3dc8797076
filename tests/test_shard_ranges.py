"""Host-side logic of the partitioned multi-GPU solver (csrc/group.cuh),
on CPU: the owned ranges of a group's shards (mp_shard_range, the same rule
group_ranges applies) tile the scene -- contiguous, disjoint, aligned to
level-1 aggregates (whole subdomains, whole aggregates: mas.py:63-77,
155-169) -- and a world_size-2 gloo job whose ranks each take their own
range agrees on the tiling (allgather)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_19892_b200 import _native


@pytest.mark.parametrize("n,bs,levels,cb", [(46664, 32, 2, 4), (12, 32, 2, 4), (202589, 32, 2, 4),
                                             (1140000, 32, 2, 32), (1000, 8, 0, 4), (999, 32, 1, 3)])
@pytest.mark.parametrize("nshards", [1, 2, 3, 4, 8])
def test_ranges_tile_the_scene(n, bs, levels, cb, nshards):
    rs = [_native.shard_range(n, bs, levels, cb, r, nshards) for r in range(nshards)]
    D = -(-n // bs)
    coarse = levels >= 1 and -(-D // cb) != D
    unit = bs * cb if coarse else bs
    assert rs[0]["verts"][0] == 0 and rs[-1]["verts"][1] == n
    assert rs[0]["subdomains"][0] == 0 and rs[-1]["subdomains"][1] == D
    for a, b in zip(rs, rs[1:]):
        assert a["verts"][1] == b["verts"][0] and a["chunks"][1] == b["chunks"][0]
        assert a["subdomains"][1] == b["subdomains"][0] or a["verts"][0] == a["verts"][1]
    for r in rs:
        v0, v1 = r["verts"]
        assert v0 % unit == 0 and (v1 % unit == 0 or v1 == n)   # whole aggregates
        assert r["subdomains"] == (v0 // bs, -(-v1 // bs))
        if coarse:
            assert r["aggregates"] == r["chunks"]
    sizes = [r["chunks"][1] - r["chunks"][0] for r in rs]
    assert max(sizes) - min(sizes) <= 1  # balanced


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    r = _native.shard_range(46664, 32, 2, 4, rank, ws)
    mine = torch.tensor([r["verts"][0], r["verts"][1], r["chunks"][0], r["chunks"][1]], dtype=torch.int64)
    allr = [torch.zeros_like(mine) for _ in range(ws)]
    dist.all_gather(allr, mine)
    out[rank] = np.stack([a.numpy() for a in allr]).tolist()
    dist.destroy_process_group()


def test_two_rank_gloo_tiling():
    ws = 2
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
        res = dict(out)
    assert res[0] == res[1]
    t = np.array(res[0])
    assert t[0, 0] == 0 and t[-1, 1] == 46664 and t[0, 1] == t[1, 0] and t[0, 3] == t[1, 2] == 182 and t[1, 3] == 365
