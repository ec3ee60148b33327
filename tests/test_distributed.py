"""Multi-rank host logic on CPU (gloo, world_size 2): view sharding and the
max-over-ranks timing reduction used by bench.py under torchrun."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_17712_b200 import distributed as fd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_view_shard_partitions_contiguously():
    for n in (0, 1, 7, 64, 65):
        for w in (1, 2, 3, 4, 8):
            shards = [fd.view_shard(n, r, w) for r in range(w)]
            flat = [v for s in shards for v in s]
            assert flat == list(range(n))
            sizes = [len(s) for s in shards]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        fd.view_shard(10, 2, 2)


def test_step_views_weak_scaling():
    a = fd.step_views(8, 0)
    b = fd.step_views(8, 1)
    assert a == list(range(8)) and b == list(range(8, 16))
    assert fd.step_views(40, 1) == [(40 + s) % 64 for s in range(40)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = fd.world()
    views = fd.view_shard(64, r, w)
    # a stand-in engine: the "frame" returns the view index (no GPU on this host)
    res = fd.run_views(lambda: object(), views, lambda eng, v: v)
    t = fd.max_over_ranks([1.0 + r, 10.0 - r])
    fd.barrier()
    gathered = [None] * w
    dist.all_gather_object(gathered, res)
    dist.destroy_process_group()
    q.put((r, t, gathered))


def test_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, t, gathered in out:
        assert t == [2.0, 10.0]  # element-wise max over ranks
        assert [v for shard in gathered for v in shard] == list(range(64))
