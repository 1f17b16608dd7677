"""Row-strip partitioned inpainting solve.

The north_star's layout for large images on several B200s: the finest
``La`` levels of the multigrid-ORAS hierarchy (solver.py:200-372) are cut
into P horizontal strips; each strip computes its owned rows widened by a
48-row halo, exchanges halos every smoothing sweep and combines residual
norms as partition-independent row-band partials (so every P gives the
bit-identical solve); the coarse levels are agglomerated (replicated).  See
csrc/strips.cu for the kernels and the transport.

Transports:
* one process holding all P strips on one GPU (``StripSolver(..., strips=P)``)
  -- device copies; the single-GPU harness that proves P-independence;
* one strip per rank over NCCL (``StripSolver.distributed(...)`` inside a
  ``torch.distributed`` job, one process per GPU): point-to-point halo
  sends/receives, an all-reduce of zero-padded band sums, broadcasts for the
  agglomeration gather -- NVLink / NVSwitch on a B200 box.

The plan (which rows each strip owns at each level) is pure host arithmetic
(``strip_plan``) and is what the multi-process CPU tests exercise.
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np
import torch

from . import _lib
from ._lib import SolveReport as _CReport
from ._lib import call, ptr, stream
from .grid import Image, Mask
from .solver import MultigridConfig, SolverReport, _enforce, _masked_rhs

HALO = 48   # rows: >= ORAS block (32) + stencil (1), a multiple of BAND
BAND = 16   # rows per residual-norm band (csrc/mgfast.cu MRB)


def level_dims(height, width, cfg: MultigridConfig | None = None):
    """Level sizes of the hierarchy (solver.py:238-243): halve (ceil) until
    max(h, w) <= block, or `levels` levels."""
    cfg = cfg or MultigridConfig()
    dims, h, w = [], height, width
    while True:
        dims.append((h, w))
        if cfg.levels > 0:
            if len(dims) >= cfg.levels or max(h, w) <= 2:
                break
        elif max(h, w) <= cfg.oras.block:
            break
        h, w = (h + 1) // 2, (w + 1) // 2
    return dims


def _feasible(dims, P, La, halo):
    if La >= len(dims):
        return False
    for lv in range(La):
        h, w = dims[lv]
        if w % 4 or w < 128:
            return False
    if La == 0 or P == 1:
        return True
    align = BAND << (La - 1)
    H = dims[0][0]
    bounds = [0] + [int(round(p * H / P / align)) * align for p in range(1, P)] + [H]
    for lv in range(La):
        hl = dims[lv][0]
        for p in range(P):
            a = bounds[p] >> lv
            b = hl if p == P - 1 else bounds[p + 1] >> lv
            if b - a < halo:
                return False
    return True


def max_partitioned_levels(height, width, P, cfg=None, halo=HALO):
    dims = level_dims(height, width, cfg)
    best = 0
    for La in range(1, len(dims)):
        if _feasible(dims, P, La, halo):
            best = La
    return best


def strip_plan(height, width, P, La=None, cfg=None, halo=HALO):
    """Owned rows of every strip at every partitioned level.

    Returns ``(La, o0, o1)`` with ``o0[lv][p]`` / ``o1[lv][p]``.  Strip
    boundaries are multiples of ``16 * 2**(La-1)`` rows, so every partitioned
    level cuts on a 16-row norm band; every strip owns >= ``halo`` rows at
    every partitioned level (a halo then comes from the adjacent strip only).
    """
    dims = level_dims(height, width, cfg)
    if La is None:
        La = max_partitioned_levels(height, width, P, cfg, halo)
    if La > 0 and not _feasible(dims, P, La, halo):
        raise ValueError(f"{P} strips of {height}x{width} cannot partition {La} levels")
    o0 = [[0] * P for _ in range(La)]
    o1 = [[0] * P for _ in range(La)]
    if La == 0:
        return 0, o0, o1
    align = BAND << (La - 1)
    bounds = [0] + [int(round(p * height / P / align)) * align for p in range(1, P)] + [height]
    for lv in range(La):
        hl = dims[lv][0]
        for p in range(P):
            o0[lv][p] = bounds[p] >> lv
            o1[lv][p] = hl if p == P - 1 else bounds[p + 1] >> lv
    return La, o0, o1


def halo_ranges(o0, o1, lv, p, level_height, halo=HALO):
    """(recv, send) row ranges of strip p at level lv: recv = {q: (r0, r1)}
    rows it takes from neighbour q, send = {q: (s0, s1)} rows q takes from
    it (the same rule as csrc/strips.cu exchange())."""
    P = len(o0[lv])
    a, b = o0[lv][p], o1[lv][p]
    e0, e1 = max(0, a - halo), min(level_height, b + halo)
    recv, send = {}, {}
    if p > 0:
        recv[p - 1] = (e0, a)
        send[p - 1] = (b_prev := o1[lv][p - 1], min(level_height, b_prev + halo))
    if p < P - 1:
        recv[p + 1] = (b, e1)
        send[p + 1] = (max(0, o0[lv][p + 1] - halo), o0[lv][p + 1])
    return recv, send


class NcclComm:
    """An NCCL communicator of the library (csrc/strips.cu), bootstrapped over
    an initialised ``torch.distributed`` group (rank 0's unique id is
    broadcast as a Python object)."""

    def __init__(self):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("NcclComm needs torch.distributed to be initialised")
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            call("sp_nccl_unique_id", uid)
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        self._c = ctypes.c_void_p()
        call("sp_nccl_comm_create", ctypes.byref(self._c), uid, self.world, self.rank)

    @property
    def handle(self):
        return self._c

    def close(self):
        if self._c:
            _lib.load().sp_nccl_comm_destroy(self._c)
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_SENDRECV = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                             ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t)
_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                          ctypes.c_int)


def _host_view(addr, nbytes, dtype=torch.uint8):
    """A CPU tensor over `nbytes` of (pinned) host memory at `addr`."""
    if nbytes == 0:
        return torch.empty(0, dtype=dtype)
    buf = (ctypes.c_uint8 * nbytes).from_address(addr)
    return torch.frombuffer(buf, dtype=torch.uint8).view(dtype)


class HostComm:
    """Host-staged strip transport over the current ``torch.distributed``
    group (any backend with CPU point-to-point, e.g. gloo): the library hands
    pinned host buffers to these callbacks (sp_strip_set_host_transport).
    It runs the multi-rank strip protocol where NCCL cannot -- several ranks
    sharing one GPU (the CI harness) -- at host-copy speed; NcclComm is the
    performance transport."""

    def __init__(self):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("HostComm needs torch.distributed to be initialised")
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.calls = {"sendrecv": 0, "allreduce": 0, "bcast": 0}
        self._cbs = (_SENDRECV(self._sendrecv), _ALLREDUCE(self._allreduce), _BCAST(self._bcast))

    def _sendrecv(self, user, peer, sp_, sb, rp, rb):
        try:
            reqs = []
            if sb:
                reqs.append(self.dist.isend(_host_view(sp_, sb), peer))
            if rb:
                reqs.append(self.dist.irecv(_host_view(rp, rb), peer))
            for q in reqs:
                q.wait()
            self.calls["sendrecv"] += 1
            return 0
        except Exception:
            return -1

    def _allreduce(self, user, p, n):
        try:
            self.dist.all_reduce(_host_view(p, 8 * n, torch.float64))
            self.calls["allreduce"] += 1
            return 0
        except Exception:
            return -1

    def _bcast(self, user, p, nbytes, root):
        try:
            self.dist.broadcast(_host_view(p, nbytes), root)
            self.calls["bcast"] += 1
            return 0
        except Exception:
            return -1

    def install(self, group_handle):
        f = [ctypes.cast(cb, ctypes.c_void_p) for cb in self._cbs]
        call("sp_strip_set_host_transport", group_handle, f[0], f[1], f[2], None)

    def close(self):
        pass


class _StripGroup:
    """One native strip group (csrc/strips.cu): P strips of a (C, H, W)
    float32 hierarchy, the strips [first, first + nloc) held here."""

    def __init__(self, key, comm):
        C, H, W, block, overlap, levels, pre, post, alpha, rho, P, La, nloc, first = key[:14]
        self.key = key
        self.La, self.o0, self.o1 = strip_plan(H, W, P, La, _cfg_of(key))
        flat0 = np.array([v for row in self.o0 for v in row] or [0], np.int32)
        flat1 = np.array([v for row in self.o1 for v in row] or [0], np.int32)
        self.h = ctypes.c_void_p()
        nccl = comm is not None and not isinstance(comm, HostComm)
        call("sp_strip_create", ctypes.byref(self.h), C, H, W, block, overlap, levels, pre,
             post, alpha, rho, P, nloc, first, self.La, HALO, ptr(flat0), ptr(flat1),
             comm.handle if nccl else None)
        if isinstance(comm, HostComm):
            comm.install(self.h)
        self.has_values = False

    def destroy(self):
        if self.h:
            _lib.load().sp_strip_destroy(self.h)
            self.h = ctypes.c_void_p()


def _cfg_of(key):
    from .solver import OrasConfig
    C, H, W, block, overlap, levels, pre, post, alpha, rho = key[:10]
    return MultigridConfig(levels=levels, pre=pre, post=post,
                           oras=OrasConfig(block=block, overlap=overlap, alpha=alpha, rho=rho))


class _GroupPool:
    """Free strip groups, least-recently released first out (a group owns P
    full-size hierarchies, so they are reused across solves and pipeline
    runs).  At most `keep` per key and `max_total` overall stay resident;
    `clear()` returns them all to the device."""

    def __init__(self, keep=2, max_total=4):
        self.keep = keep
        self.max_total = max_total
        self.free = []                      # oldest first

    def acquire(self, key, comm):
        for i in range(len(self.free) - 1, -1, -1):
            if self.free[i].key == key:
                return self.free.pop(i)
        return _StripGroup(key, comm)

    def release(self, g):
        same = [x for x in self.free if x.key == g.key]
        if len(same) >= self.keep:
            self.free.remove(same[0])
            same[0].destroy()
        self.free.append(g)
        while len(self.free) > self.max_total:
            self.free.pop(0).destroy()

    def __len__(self):
        return len(self.free)

    def clear(self):
        for g in self.free:
            g.destroy()
        self.free.clear()


_GPOOL = _GroupPool()


class StripHierarchy:
    """`GridHierarchy` on a strip group: the mask (and stored-value) pyramid
    of one mask and `solve_sym` (solver.py:328-372) over the strips."""

    def __init__(self, owner: "StripSolver", mask_t, values_t):
        self.owner = owner
        H, W = mask_t.shape
        self.mask_t = mask_t
        self.channels = owner.channels
        self.height, self.width = H, W
        self.cfg = owner.cfg
        self._g = _GPOOL.acquire(owner._key, owner._comm)
        call("sp_strip_set_mask", self._g.h, ptr(mask_t), ptr(values_t), stream())
        self.has_values = values_t is not None
        self._rep = _CReport()

    def __del__(self):
        g = getattr(self, "_g", None)
        if g is not None:
            try:
                _GPOOL.release(g)
            except Exception:
                pass
            self._g = None

    @property
    def nlevels(self):
        n = ctypes.c_int()
        dims = (ctypes.c_int * 128)()
        call("sp_strip_levels", self._g.h, ctypes.byref(n), dims, 128)
        return n.value

    def solve_sym(self, bsym, init=None, tol=None, cycles=None, max_cycles=None,
                  cascade=False, values=False):
        cfg = self.cfg
        t0 = time.perf_counter()
        b = bsym.to(torch.float32).contiguous()
        if values:  # stored values x -> b~ = sym_rhs(where(mask, x, 0))
            b = _masked_rhs(b, self.mask_t)
        if init is not None:
            u = init.to(torch.float32).clone()
            mode = 1
        else:
            u = torch.empty_like(b)
            mode = 2 if (cascade and self.has_values) else 0
            if cascade and not self.has_values and self.nlevels > 1:
                raise ValueError("hierarchy was built without stored values")
        rep = self._rep
        call("sp_strip_solve", self._g.h, ptr(b), ptr(u), mode,
             -1.0 if tol is None else float(tol),
             int(cfg.cycles if cycles is None else cycles),
             int(cfg.max_cycles if max_cycles is None else max_cycles), ctypes.byref(rep),
             stream())
        out = SolverReport(iterations=rep.iterations, converged=bool(rep.converged),
                           residuals=[rep.residuals[i] for i in range(rep.nres)])
        out.seconds = time.perf_counter() - t0
        return u, out


class StripSolver:
    """`InpaintSolver` (solver.py:514-536) on a row-strip partition.

    ``StripSolver(h, w, c, strips=P)``: all P strips in this process (one
    GPU).  ``StripSolver.distributed(h, w, c)``: one strip per rank of the
    current ``torch.distributed`` job, NCCL transport.  float32 only.  Every
    rank returns the gathered (full) solution, bit-identical for every P.
    It can stand in for the `InpaintSolver` of the pipeline stages
    (`delaunay_densify`, the tonal optimizers, `run_pipeline(...,
    solver=...)`): `inpaint` and `hierarchy` follow `InpaintSolver`.
    """

    def __init__(self, height, width, channels, strips=1, cfg: MultigridConfig | None = None,
                 La=None, _rank=None, _comm=None):
        self.cfg = cfg if cfg is not None else MultigridConfig()
        if self.cfg.dtype != "float32":
            raise ValueError("the strip solver runs float32")
        self.height, self.width, self.channels = height, width, channels
        self.P = strips
        self.La, self.o0, self.o1 = strip_plan(height, width, strips, La, self.cfg)
        nloc, first = (strips, 0) if _rank is None else (1, _rank)
        self.rank = 0 if _rank is None else _rank
        self._comm = _comm
        o = self.cfg.oras
        self._key = (channels, height, width, o.block, o.overlap, self.cfg.levels, self.cfg.pre,
                     self.cfg.post, float(o.alpha), float(o.rho), strips, self.La, nloc, first,
                     id(_comm) if _comm is not None else 0)

    @classmethod
    def distributed(cls, height, width, channels, cfg=None, La=None, transport="nccl"):
        """One strip per rank of the current ``torch.distributed`` job.
        transport "nccl": the library's NCCL communicator (one GPU per rank);
        "host": host-staged exchanges through torch.distributed (HostComm --
        e.g. gloo ranks sharing one GPU)."""
        import torch.distributed as dist
        if transport not in ("nccl", "host"):
            raise ValueError("transport must be 'nccl' or 'host'")
        comm = NcclComm() if transport == "nccl" else HostComm()
        return cls(height, width, channels, strips=dist.get_world_size(), cfg=cfg, La=La,
                   _rank=dist.get_rank(), _comm=comm)

    @property
    def distributed_ranks(self):
        return self.P if self._comm is not None else 1

    def strip_geometry(self, ws):
        """The densification geometry partitioned by this solver's row
        strips (geometry.StripGeometry) when it spans several ranks, else
        None (the workspace runs whole)."""
        if self._comm is None or self.P < 2:
            return None
        from .geometry import DistGather, StripGeometry
        rows = [(self.o0[0][p], self.o1[0][p]) for p in range(self.P)] if self.La else \
            [(self.height * p // self.P, self.height * (p + 1) // self.P) for p in range(self.P)]
        self.geometry = StripGeometry(ws, rows, self.rank, DistGather())
        return self.geometry

    def _check(self, shape):
        if tuple(shape) != (self.height, self.width):
            raise ValueError("image does not match the strip solver's geometry")

    def hierarchy(self, mask: Mask, values: Image | None = None, channels=None):
        m_t = mask.tensor()
        self._check(m_t.shape)
        v = None if values is None else values.tensor(torch.float32)
        return StripHierarchy(self, m_t, v)

    def inpaint(self, f: Image, mask: Mask, init: Image | None = None, tol=-1.0, cycles=None):
        """solver.py:485-511 on the strips: FMG cascade unless `init`; the
        result interpolates f exactly on the mask (gathered on every rank)."""
        cfg = self.cfg
        tol = cfg.tol if tol == -1.0 else tol
        if mask.count == 0:
            raise ValueError("singular system: empty mask")
        t0 = time.perf_counter()
        f_t = f.tensor(torch.float32)
        m_t = mask.tensor()
        if tuple(f_t.shape) != (self.channels, self.height, self.width):
            raise ValueError("image does not match the strip solver's geometry")
        hier = StripHierarchy(self, m_t, f_t)
        bsym = _masked_rhs(f_t, m_t)
        init_t = None if init is None else init.tensor(torch.float32)
        u, out = hier.solve_sym(bsym, init=init_t, tol=tol, cycles=cycles,
                                cascade=cfg.mode == "fmg" and init is None)
        _enforce(u, f_t, m_t)
        out.seconds = time.perf_counter() - t0
        return Image(u), out
