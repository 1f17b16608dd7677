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
