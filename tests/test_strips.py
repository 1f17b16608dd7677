"""Host logic of the row-strip partitioned solve on CPU.

* the strip plan: alignment, coverage and halo invariants that
  csrc/strips.cu relies on (and validates again at creation);
* the transport protocol with real collectives: world_size 2 and 3 gloo
  processes (one strip per rank, as under torchrun with NCCL on a B200 box)
  run the halo exchange of `halo_ranges`, the zero-padded band-sum
  all-reduce (bit-exact gather) and the agglomeration broadcasts, and check
  every rank ends with the rows of the single-process image.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2401_06747_b200.strips import (BAND, HALO, halo_ranges, level_dims,  # noqa: E402
                                          max_partitioned_levels, strip_plan)


@pytest.mark.parametrize("H,W", [(2160, 3840), (4320, 7680), (1024, 1536), (517, 640),
                                 (301, 512), (96, 4096)])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_plan_invariants(H, W, P):
    dims = level_dims(H, W)
    La, o0, o1 = strip_plan(H, W, P)
    assert La == max_partitioned_levels(H, W, P)
    assert La < len(dims)
    for lv in range(La):
        hl, wl = dims[lv]
        assert wl % 4 == 0 and wl >= 128
        assert o0[lv][0] == 0 and o1[lv][P - 1] == hl
        for p in range(P):
            assert o0[lv][p] % BAND == 0
            assert o1[lv][p] % BAND == 0 or p == P - 1
            if p:
                assert o0[lv][p] == o1[lv][p - 1]
            if P > 1:
                assert o1[lv][p] - o0[lv][p] >= HALO
            if lv:  # coarse owned rows are the restriction of the fine ones
                assert o0[lv][p] * 2 == o0[lv - 1][p]
    if La:
        with pytest.raises(ValueError):
            strip_plan(H, W, P, La=len(dims))


def test_plan_uses_deeper_partition_for_fewer_strips():
    las = [max_partitioned_levels(4320, 7680, P) for P in (1, 2, 4, 8)]
    assert las == sorted(las, reverse=True) and las[-1] >= 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        C, H, W = 2, 640, 256
        La, o0, o1 = strip_plan(H, W, world)
        dims = level_dims(H, W)
        ok = []
        for lv in range(La):
            hl, wl = dims[lv]
            truth = torch.arange(C * hl * wl, dtype=torch.float32).reshape(C, hl, wl)
            x = torch.full_like(truth, float("nan"))
            a, b = o0[lv][rank], o1[lv][rank]
            x[:, a:b] = truth[:, a:b]
            recv, send = halo_ranges(o0, o1, lv, rank, hl)
            ops, bufs = [], {}
            for q_, (s0, s1) in send.items():
                if s1 > s0:
                    ops.append(dist.P2POp(dist.isend, x[:, s0:s1].contiguous(), q_))
            for q_, (r0, r1) in recv.items():
                if r1 > r0:
                    bufs[q_] = torch.empty((C, r1 - r0, wl))
                    ops.append(dist.P2POp(dist.irecv, bufs[q_], q_))
            for r in dist.batch_isend_irecv(ops) if ops else []:
                r.wait()
            for q_, (r0, r1) in recv.items():
                if r1 > r0:
                    x[:, r0:r1] = bufs[q_]
            e0, e1 = max(0, a - HALO), min(hl, b + HALO)
            ok.append(bool(torch.equal(x[:, e0:e1], truth[:, e0:e1])))
            # zero-padded band sums: an all-reduce SUM is an exact gather
            nb = -(-hl // BAND)
            rng = np.random.default_rng(lv)
            band_truth = torch.from_numpy(rng.random((C, nb)))
            mine = torch.zeros_like(band_truth)
            mine[:, a // BAND:-(-b // BAND)] = band_truth[:, a // BAND:-(-b // BAND)]
            dist.all_reduce(mine)
            ok.append(bool(torch.equal(mine, band_truth)))
            tot = [float(sum(band_truth[c, i].item() for i in range(nb))) for c in range(C)]
            got = [float(sum(mine[c, i].item() for i in range(nb))) for c in range(C)]
            ok.append(tot == got)
            # agglomeration gather: every strip broadcasts its owned rows
            y = torch.full_like(truth, float("nan"))
            y[:, a:b] = truth[:, a:b]
            for p in range(world):
                pa, pb = o0[lv][p], o1[lv][p]
                buf = y[:, pa:pb].contiguous()
                dist.broadcast(buf, src=p)
                y[:, pa:pb] = buf
            ok.append(bool(torch.equal(y, truth)))
        q.put((rank, La, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_transport_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(r[1] >= 1 for r in res)
    assert all(all(r[2]) for r in res), res
