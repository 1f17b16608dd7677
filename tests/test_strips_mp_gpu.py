"""The multi-rank strip path EXECUTED: two processes (torch.distributed,
gloo) share the one GPU, each owning one row strip of the image through
`StripSolver.distributed(..., transport="host")` -- the library's own
per-rank strip code (csrc/strips.cu: views, halo exchange, band-norm
combine, agglomeration gather, distributed RAS block sharding in tonal.py)
with the exchanges staged through host memory instead of NCCL (NCCL cannot
put two ranks on one device).  The result must be bit-identical to the
single-process solve with the same strip plan (P = 1 strips, the loopback
path), which test_strips_gpu.py already ties to every other P."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, job, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    try:
        if job == "solve":
            c, h, w = 3, 1024, 1536
            f = O.synth(h, w, c, 0)
            mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
            cfg = sp.MultigridConfig(tol=1e-6, max_cycles=60)
            s = StripSolver.distributed(h, w, c, cfg=cfg, La=2, transport="host")
            u, rep = s.inpaint(sp.Image(f), sp.Mask(mask))
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u.data,
                     res=np.array(rep.residuals), it=rep.iterations,
                     calls=np.array([s._comm.calls[k] for k in ("sendrecv", "allreduce",
                                                                "bcast")]))
        else:
            c, h, w = 3, 512, 768
            f = O.synth(h, w, c, 4)
            cfg = sp.PipelineConfig(iterations=4)
            s = StripSolver.distributed(h, w, c, cfg=cfg.solver().cfg, La=1, transport="host")
            mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg, solver=s)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), m=mask.indicator, g=st.g.data,
                     mse=st.mse, hist=np.array([r[2] for r in hist]),
                     geo_calls=s.geometry.calls)
    finally:
        dist.destroy_process_group()


def _run(job, tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(2, _port(), job, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    return [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in (0, 1)]


def test_two_rank_strip_solve_bit_identical(tmp_path):
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    r0, r1 = _run("solve", tmp_path)
    # every rank holds the gathered solution
    assert np.array_equal(r0["u"], r1["u"])
    # the exchanges really crossed the process boundary
    assert (r0["calls"] > 0).all() and (r1["calls"] > 0).all()
    c, h, w = 3, 1024, 1536
    f = O.synth(h, w, c, 0)
    mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
    cfg = sp.MultigridConfig(tol=1e-6, max_cycles=60)
    u1, rep1 = StripSolver(h, w, c, strips=1, cfg=cfg, La=2).inpaint(sp.Image(f),
                                                                    sp.Mask(mask))
    assert np.array_equal(r0["u"], u1.data)
    assert int(r0["it"]) == rep1.iterations
    assert list(r0["res"]) == rep1.residuals
    assert rep1.converged


def test_two_rank_pipeline_on_strips(tmp_path):
    """run_pipeline on a 2-rank strip solver: distributed solves, the
    densification's Delaunay step and accumulate partitioned by the strips
    (geometry.StripGeometry), and the RAS block problems sharded by rank and
    all-gathered (tonal.py gather_all) -- bit-identical to one process."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    r0, r1 = _run("pipeline", tmp_path)
    for k in ("m", "g", "hist"):
        assert np.array_equal(r0[k], r1[k])
    # the Delaunay step and the accumulate ran partitioned by the row strips
    # (geometry.StripGeometry: 2 calls per densification iteration)
    assert int(r0["geo_calls"]) > 0 and int(r1["geo_calls"]) > 0
    c, h, w = 3, 512, 768
    f = O.synth(h, w, c, 4)
    cfg = sp.PipelineConfig(iterations=4)
    s1 = StripSolver(h, w, c, strips=1, cfg=cfg.solver().cfg, La=1)
    mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg, solver=s1)
    assert np.array_equal(r0["m"], mask.indicator)
    assert np.array_equal(r0["g"], st.g.data)
    assert float(r0["mse"]) == st.mse


def _nccl_worker(_i, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    try:
        c, h, w = 3, 512, 768
        f = O.synth(h, w, c, 2)
        mask = (np.random.default_rng(3).random((h, w)) < 0.05).astype(np.uint8)
        s = StripSolver.distributed(h, w, c, transport="nccl")
        u, rep = s.inpaint(sp.Image(f), sp.Mask(mask))
        np.savez(os.path.join(out_dir, "nccl.npz"), u=u.data, it=rep.iterations,
                 handle=int(bool(s._comm.handle.value)))
        s._comm.close()
    finally:
        dist.destroy_process_group()


def test_nccl_bootstrap_single_rank(tmp_path):
    """The NCCL transport's bootstrap executes on the one GPU: libnccl.so.2
    dlopen'd by the library, rank 0's unique id broadcast through
    torch.distributed (nccl backend, world size 1), the communicator created
    and destroyed around a StripSolver.distributed solve; the result equals
    the in-process P = 1 strip solve.  (Two NCCL ranks cannot share a GPU:
    the multi-rank exchanges run under the host-staged transport above.)"""
    import torch.multiprocessing as mp
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    mp.start_processes(_nccl_worker, args=(_port(), str(tmp_path)), nprocs=1, join=True,
                       start_method="spawn")
    r = np.load(os.path.join(tmp_path, "nccl.npz"))
    assert int(r["handle"]) == 1
    c, h, w = 3, 512, 768
    f = O.synth(h, w, c, 2)
    mask = (np.random.default_rng(3).random((h, w)) < 0.05).astype(np.uint8)
    u1, rep1 = StripSolver(h, w, c, strips=1).inpaint(sp.Image(f), sp.Mask(mask))
    assert np.array_equal(r["u"], u1.data)
    assert int(r["it"]) == rep1.iterations
