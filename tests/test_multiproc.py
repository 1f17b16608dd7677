"""N>1 host logic of bench.py on CPU: world_size-2 gloo processes run the
replica bookkeeping (rank env, barrier, max over ranks) that the torchrun
launch uses on the GPU box with NCCL.  The data path has no collective
(one image per rank), so the only cross-rank traffic is the timing max."""

import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bench._barrier(world)
        got = bench._max_over_ranks(10.0 + rank, world, device="cpu")
        # each rank owns one replica image, seeded by its rank
        from oracle.oracle import synth
        img = synth(8, 8, 3, seed=rank)
        q.put((rank, got, float(img.sum())))
    finally:
        dist.destroy_process_group()


def test_replica_timing_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert [r[1] for r in res] == [11.0, 11.0]
    # replicas work on different images
    assert res[0][2] != res[1][2]


def test_reference_arm_rank_nonzero_exits_without_work(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    assert bench.main(["--impl", "reference", "--gpus", "2", "--steps", "1",
                       "--warmup", "0"]) == 0
    assert capsys.readouterr().out == ""


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # geometry.DistGather: the strip geometry's variable-length all-gather
        # (triangle keys, assignment rows, bucket ranges) under gloo
        from paper_2401_06747_b200.geometry import DistGather
        g = DistGather()
        keys = torch.arange(rank * 10, rank * 10 + 3 + 2 * rank, dtype=torch.int64)
        got = g.allgather_var(keys)
        rows = torch.full((2 + rank, 4), rank, dtype=torch.int32)
        got_rows = g.allgather_var(rows)
        buck = torch.stack([torch.tensor([1.5 + rank], dtype=torch.float64),
                            torch.tensor([7], dtype=torch.int64).view(torch.float64),
                            torch.tensor([0.25], dtype=torch.float64)])
        got_b = g.allgather_var(buck)
        q.put((rank, [t.tolist() for t in got], [tuple(t.shape) for t in got_rows],
               [t.view(3, -1)[1].contiguous().view(torch.int64).tolist() for t in got_b]))
    finally:
        dist.destroy_process_group()


def test_strip_geometry_gather_gloo():
    """The strip geometry's exchange (geometry.DistGather.allgather_var) on
    two gloo ranks: ragged key lists, ragged row blocks and bit-cast int64
    bucket argmaxes come back complete and in rank order on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    for _, keys, shapes, amax in res:
        assert keys == [[0, 1, 2], [10, 11, 12, 13, 14]]
        assert shapes == [(8,), (12,)]
        assert amax == [[7], [7]]
