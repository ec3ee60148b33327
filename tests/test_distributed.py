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


# --------------------------------------------- bench.main's rank path (gloo) ---
def _stand_in_measure(args, rank, world, local, view_ids):
    """Stands in for bench.measure_gpu (no GPU here): rank r's device time is
    10 + r ms for its views."""
    n = len(view_ids)
    return dict(views=n, dev_ms=10.0 + rank, lat_ms=0.3 * n, e2e={"compact": (12.0 + rank, 1000.0),
                                                                    "dense": (14.0, 2000.0)},
                stats=[(170000, 960)] * n, stage_ms={"depth pass": 0.1, "uv": 0.01}, clocks={"sm_mhz": None},
                launches_per_frame=25, T=1000040, V=500302, W=1920, H=1080, view_ids=list(view_ids))


def _bench_worker(rank, world, port, argv, q):
    import contextlib
    import io
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), FA_BENCH_BACKEND="gloo")
    import bench
    seen = []

    def measure(args, r, w, local, view_ids):
        seen.extend(view_ids)
        return _stand_in_measure(args, r, w, local, view_ids)

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        bench.main(argv, measure=measure)
    q.put((rank, buf.getvalue(), seen))


def _run_bench_ranks(argv, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, argv, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_bench_main_two_ranks_weak():
    import json
    out = _run_bench_ranks(["--gpus", "2", "--steps", "8", "--no-cpu-baseline"])
    (r0, text0, v0), (r1, text1, v1) = out
    assert text1 == ""  # only rank 0 prints
    lines = [ln for ln in text0.splitlines() if ln.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert v0 == list(range(8)) and v1 == list(range(8, 16))
    # all ranks' views over the max-over-ranks device time (rank 1: 11 ms)
    assert line["value"] == pytest.approx(16 / 11e-3)
    assert line["e2e"]["value"] == pytest.approx(16 / 13e-3)
    assert line["config"]["parallelism"].startswith("2 independent view streams")


def test_bench_main_two_ranks_strong_split():
    import json
    out = _run_bench_ranks(["--gpus", "2", "--split", "strong", "--no-cpu-baseline"])
    (_, text0, v0), (_, _, v1) = out
    line = json.loads(text0.strip())
    assert v0 == list(range(32)) and v1 == list(range(32, 64))
    assert line["scaling"] == "strong" and line["detail"]["views_total"] == 64
    assert line["value"] == pytest.approx(64 / 11e-3)


def test_bench_torchrun_command():
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    import bench
    cmd = bench.torchrun_cmd(["--gpus", "4", "--steps", "8"], 4, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "4", "--steps", "8"][-3:]


def test_bench_reference_config_matches_b200_arm():
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    import bench
    a = bench.parse_args(["--gpus", "1", "--steps", "20"])
    b = bench.parse_args(["--gpus", "1", "--steps", "20", "--impl", "reference"])
    assert bench.bench_config(a, 1) == bench.bench_config(b, 1)
