"""Tonal optimization: which values to store (tonal.py parity).

Mirrors /root/reference/pkg/src/sparsepaint/tonal.py:29-507 on the device.
Every matrix-free product B x / B^T y is a device multigrid solve
(GridHierarchy).  The RAS block-local normal equations (tonal.py:267-294,
343-381) are solved for ALL 64x64 blocks at once: the blocks become the
tiles of one batched hierarchy (csrc/solver.cu), the block CG bookkeeping is
kept per (tile, channel) on the device, and the blocks leave the batch
individually when their own stopping rule fires -- the same per-block
decisions the reference takes block after block.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, dcode, ptr, stream
from .geometry import VoronoiLabels, workspace
from .grid import Image, Mask
from .solver import (GridHierarchy, InpaintSolver, MultigridConfig, _enforce, _masked_rhs,
                     _starts)
from .vec import chan_dot as _chan_dot_t
from .vec import mse_t


@dataclass
class TonalState:
    """tonal.py:29-43."""

    g: Image
    u: Image
    mse: float
    history: list = field(default_factory=list)
    iterations: int = 0
    inner_solves: int = 0
    converged: bool = True

    @property
    def psnr(self) -> float:
        return math.inf if self.mse == 0 else 10 * math.log10(255.0 ** 2 / self.mse)


@dataclass
class RasTonalConfig:
    """tonal.py:46-64."""

    block: int = 64
    overlap: int = 6
    local_iters: int = 30
    local_tol: float = 0.1
    inner_cycles: int = 2
    inner_tol: float | None = None
    cold_tol: float = 1e-4
    local_product_tol: float = 1e-2
    rel_improvement: float = 1e-3
    max_outer: int = 50
    final_tol: float = 1e-6

    def __post_init__(self):
        if self.block < self.overlap + 2:
            raise ValueError("block size must be at least overlap + 2")
        if self.local_iters < 1 or self.max_outer < 1:
            raise ValueError("iteration caps must be positive")


@dataclass
class InitConfig:
    """tonal.py:67-83."""

    scheme: str = "voronoi-richardson"
    tau: float = 1.0
    weight_scheme: str = "inverse-log"
    max_steps: int = 20
    stop_on_mse_increase: bool = True
    inner_cycles: int = 2
    inner_tol: float | None = None
    final_tol: float = 1e-6

    def __post_init__(self):
        if self.tau <= 0:
            raise ValueError("step size must be positive")
        if self.scheme not in ("none", "neighbor-balance", "voronoi-richardson"):
            raise ValueError("unknown initialization scheme")


def _where_mask(x, m_t):
    out = torch.empty_like(x)
    C, H, W = x.shape
    call("sp_where_mask", dcode(x), ptr(x), ptr(m_t), ptr(out), C, H, W, stream())
    return out


def _ct_apply(w, m_t):
    out = torch.empty_like(w)
    C, H, W = w.shape
    call("sp_ct_apply", dcode(w), ptr(w), ptr(m_t), ptr(out), C, H, W, 1.0, stream())
    return out


class _TonalSystem:
    """tonal.py:100-144: matrix-free B / B^T on one mask (device)."""

    def __init__(self, mask_t, solver: InpaintSolver, channels, inner_cycles=1,
                 inner_tol=None, cold_tol=1e-4, cold_max_cycles=100):
        self.mask = mask_t
        # the solver's own hierarchy type (GridHierarchy, or the row-strip
        # hierarchy of strips.StripSolver)
        self.hier = solver.hierarchy(Mask(mask_t), None, channels=channels)
        self.inner_cycles = inner_cycles
        self.inner_tol = inner_tol
        self.cold_tol = cold_tol
        self.cold_max_cycles = cold_max_cycles
        self.dtype = solver.cfg.torch_dtype
        self.solves = 0

    def _solve(self, bsym, warm, tol=None, cycles=None, values=False):
        self.solves += 1
        if tol is None:
            if self.inner_tol is not None:
                tol = self.inner_tol
            elif warm is None:
                tol = self.cold_tol
        u, _ = self.hier.solve_sym(bsym, init=warm, tol=tol,
                                   cycles=self.inner_cycles if cycles is None else cycles,
                                   max_cycles=self.cold_max_cycles, values=values)
        return u

    def apply_B(self, x, warm=None, tol=None, cycles=None):
        # B x = solve(A~, C~ (mask ? x : 0)): the rhs is formed in the hierarchy
        return self._solve(x.to(self.dtype).contiguous(), warm, tol, cycles, values=True)

    def apply_Bt(self, y, warm=None, tol=None, cycles=None):
        w = self._solve(y.to(self.dtype).contiguous(), warm, tol, cycles)
        return _ct_apply(w, self.mask), w


def _f_dt(f: Image, dtype):
    return f.tensor(dtype)


def apply_B(x: Image, mask: Mask, solver: InpaintSolver | None = None,
            inner_tol: float = 1e-8) -> Image:
    """tonal.py:147-155."""
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    if solver is None:
        solver = InpaintSolver(MultigridConfig(dtype="float64"))
    xt = x.tensor(solver.cfg.torch_dtype)
    sys_ = _TonalSystem(mask.tensor(), solver, xt.shape[0], inner_tol=inner_tol)
    return Image(sys_.apply_B(xt))


def apply_Bt(y: Image, mask: Mask, solver: InpaintSolver | None = None,
             inner_tol: float = 1e-8) -> Image:
    """tonal.py:158-167."""
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    if solver is None:
        solver = InpaintSolver(MultigridConfig(dtype="float64"))
    yt = y.tensor(solver.cfg.torch_dtype)
    sys_ = _TonalSystem(mask.tensor(), solver, yt.shape[0], inner_tol=inner_tol)
    z, _ = sys_.apply_Bt(yt)
    return Image(z)


def initial_state(f: Image, mask: Mask, solver: InpaintSolver | None = None,
                  final_tol: float = 1e-6) -> TonalState:
    """tonal.py:170-180."""
    if solver is None:
        solver = InpaintSolver()
    u, rep = solver.inpaint(f, mask, tol=final_tol)
    ut = u.tensor()
    g = _where_mask(f.tensor(ut.dtype), mask.tensor())
    return TonalState(g=Image(g), u=u, mse=mse_t(f.tensor(torch.float64), ut),
                      converged=rep.converged)


def _final_state(f64, mask_t, sys_: _TonalSystem, g_best, warm, history, iterations,
                 final_tol) -> TonalState:
    """tonal.py:183-195: tight reconstruction of the best values."""
    u, rep = sys_.hier.solve_sym(g_best.to(sys_.dtype).contiguous(), init=warm, tol=final_tol,
                                 values=True)
    sys_.solves += 1
    _enforce(u, g_best.to(u.dtype).contiguous(), mask_t)
    # g is zero off the mask by construction; make it exact and let the host
    # copy move only the stored values
    g_out = _where_mask(g_best.contiguous(), mask_t)
    return TonalState(g=Image.sparse(g_out, mask_t), u=Image(u), mse=mse_t(f64, u),
                      history=history, iterations=iterations, inner_solves=sys_.solves,
                      converged=rep.converged)


def _dots(a, b):
    return _chan_dot_t(a, b).cpu().numpy()


def cgnr_tonal(f: Image, mask: Mask, init: TonalState | None = None,
               solver: InpaintSolver | None = None, rel_improvement: float = 1e-3,
               max_iters: int = 100, inner_cycles: int = 1, inner_tol: float | None = None,
               cold_tol: float = 1e-4, final_tol: float = 1e-6) -> TonalState:
    """tonal.py:198-264: CG on the normal equations (per-channel alpha/beta,
    dots in double, MSE from the primal residual, best iterate)."""
    if solver is None:
        solver = InpaintSolver()
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    m_t = mask.tensor()
    dt = solver.cfg.torch_dtype
    f64 = f.tensor(torch.float64)
    f_arr = f64.to(dt)
    C = f_arr.shape[0]
    sys_ = _TonalSystem(m_t, solver, C, inner_cycles, inner_tol, cold_tol=cold_tol)
    if init is None:
        g = _where_mask(f_arr, m_t)
        warm = None
    else:
        g = _where_mask(init.g.tensor(dt), m_t)
        warm = init.u.tensor(dt)
    npdt = np.float32 if dt == torch.float32 else np.float64
    t0 = time.perf_counter()
    history = []
    u = sys_.apply_B(g, warm=warm)
    r = f_arr - u
    mse = mse_t(f_arr, u)
    best_g, best_mse = g.clone(), mse
    history.append((0, mse, time.perf_counter() - t0, sys_.solves))
    z, w_warm = sys_.apply_Bt(r)
    zs = _dots(z, z)
    p = z.clone()
    it = 0
    prev_mse = mse
    while it < max_iters and zs.sum() > 0:
        w = sys_.apply_B(p)
        ws = _dots(w, w)
        alpha = np.where(ws > 0, zs / np.where(ws > 0, ws, 1), 0.0)
        a = torch.from_numpy(alpha.astype(npdt)).to(g.device)[:, None, None]
        g = g + a * p
        r = r - a * w
        mse = mse_t(r, torch.zeros_like(r, dtype=torch.float64))
        it += 1
        history.append((it, mse, time.perf_counter() - t0, sys_.solves))
        if mse < best_mse:
            best_mse, best_g = mse, g.clone()
        if prev_mse - mse < rel_improvement * prev_mse:
            break
        prev_mse = mse
        z, w_warm = sys_.apply_Bt(r, warm=w_warm)
        zs_new = _dots(z, z)
        beta = np.where(zs > 0, zs_new / np.where(zs > 0, zs, 1), 0.0)
        p = z + torch.from_numpy(beta.astype(npdt)).to(g.device)[:, None, None] * p
        zs = zs_new
    return _final_state(f64, m_t, sys_, best_g, u, history, it, final_tol)


# ---------------------------------------------------------------------------
# RAS: batched block-local normal-equation solves
# ---------------------------------------------------------------------------

def _cover_tables(starts, size, dim):
    """First covering block and number of covering blocks per row/column
    (sorted starts; vectorised)."""
    st = np.asarray(starts, np.int64)
    y = np.arange(dim)
    first = np.searchsorted(st + size, y, side="right")
    last = np.searchsorted(st, y, side="right") - 1
    nn = np.maximum(last - first + 1, 0).astype(np.int32)
    k0 = np.where(nn > 0, first, 0).astype(np.int32)
    return k0, nn


_RAS_GEOM: dict = {}


def _ras_geometry(H, W, bh, bw, stride, dev):
    """The mask-independent RAS block tables of an (H, W) image (block
    origins, cover tables), host and device copies, cached per geometry --
    host numpy work and uploads that every ras_tonal call repeated."""
    key = (H, W, bh, bw, stride, str(dev))
    g = _RAS_GEOM.get(key)
    if g is None:
        if len(_RAS_GEOM) > 8:
            _RAS_GEOM.clear()
        ys = _starts(H, bh, stride).astype(np.int32)
        xs = _starts(W, bw, stride).astype(np.int32)
        oy_all = np.repeat(ys, xs.size)
        ox_all = np.tile(xs, ys.size)
        rk0, rn = _cover_tables(ys, bh, H)
        ck0, cn = _cover_tables(xs, bw, W)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        g = dict(ys=ys, xs=xs, oy_all=oy_all, ox_all=ox_all, oy_t=t(oy_all), ox_t=t(ox_all),
                 ys_t=t(ys), xs_t=t(xs), rk0=t(rk0), rn=t(rn), ck0=t(ck0), cn=t(cn))
        _RAS_GEOM[key] = g
    return g


class _RasBlocks:
    """The 64x64 (block/overlap) decomposition of the tonal RAS, its
    active blocks (>= 1 stored pixel, tonal.py:349-350) as tiles of one
    batched hierarchy, and the scatter tables."""

    def __init__(self, mask_t, solver: InpaintSolver, C, cfg: RasTonalConfig):
        H, W = mask_t.shape
        dev = mask_t.device
        self.H, self.W, self.C = H, W, C
        self.bh, self.bw = min(cfg.block, H), min(cfg.block, W)
        stride = cfg.block - cfg.overlap
        geo = _ras_geometry(H, W, self.bh, self.bw, stride, dev)
        ys, xs = geo["ys"], geo["xs"]
        self.nby, self.nbx = ys.size, xs.size
        nb = self.nby * self.nbx
        oy_all, ox_all = geo["oy_all"], geo["ox_all"]
        # per-block stored-pixel counts on the device (one pass)
        oy_t, ox_t = geo["oy_t"], geo["ox_t"]
        mt_all = torch.empty((nb, self.bh, self.bw), dtype=torch.uint8, device=dev)
        call("sp_gather_mask_tiles", ptr(mask_t), ptr(oy_t), ptr(ox_t), nb, H, W, self.bh,
             self.bw, ptr(mt_all), stream())
        has = (mt_all.view(nb, -1).sum(1) > 0).cpu().numpy()
        act = np.nonzero(has)[0]
        self.nt_all = int(act.size)
        tile_of = np.full(nb, -1, np.int32)
        tile_of[act] = np.arange(self.nt_all, dtype=np.int32)
        self.tile_of = torch.from_numpy(tile_of).to(dev)
        # a distributed (multi-rank strip) solver shards the independent block
        # problems by rank; the block corrections are all-gathered before the
        # scatter, which every rank then runs over all blocks in block order
        self.ranks = getattr(solver, "distributed_ranks", 1)
        self.rank = getattr(solver, "rank", 0) if self.ranks > 1 else 0
        self.chunk = -(-self.nt_all // self.ranks)
        self.t0 = min(self.nt_all, self.rank * self.chunk)
        self.t1 = min(self.nt_all, self.t0 + self.chunk)
        act_loc = act[self.t0:self.t1]
        self.nt = int(act_loc.size)
        if self.nt == nb:
            # every block holds a stored pixel (the usual case at a few %
            # density): the cached origins and the gathered masks as they are
            self.oy, self.ox, self.tmask = oy_t, ox_t, mt_all
        else:
            self.oy = torch.from_numpy(oy_all[act_loc].copy()).to(dev)
            self.ox = torch.from_numpy(ox_all[act_loc].copy()).to(dev)
            self.tmask = (mt_all[torch.from_numpy(act_loc).to(dev)].contiguous() if self.nt
                          else mt_all[:0])
        self.ys_t, self.xs_t = geo["ys_t"], geo["xs_t"]
        self.rk0, self.rn = geo["rk0"], geo["rn"]
        self.ck0, self.cn = geo["ck0"], geo["cn"]
        self.dtype = solver.cfg.torch_dtype
        self.inner_cycles = cfg.inner_cycles
        self.tol = cfg.inner_tol if cfg.inner_tol is not None else cfg.local_product_tol
        self.solves = 0
        self.hier = None
        if self.nt:
            o = solver.cfg.oras
            key = (dcode(torch.empty(0, dtype=self.dtype)), C, self.bh, self.bw, o.block,
                   o.overlap, solver.cfg.levels, solver.cfg.pre, solver.cfg.post,
                   float(o.alpha), float(o.rho), 0, self.nt)
            from .solver import _POOL
            h = _POOL.acquire(key)
            self.hier = GridHierarchy(h, key, solver.cfg, C, self.bh, self.bw, False)
            call("sp_hier_set_mask", h, ptr(self.tmask), None, stream())
        self._iters = np.zeros(max(1, self.nt), np.int32)
        self._conv = np.zeros(max(1, self.nt), np.int32)

    def gather(self, img):
        out = torch.empty((self.nt, self.C, self.bh, self.bw), dtype=img.dtype,
                          device=img.device)
        if self.nt:
            call("sp_gather_tiles", dcode(img), ptr(img), ptr(self.oy), ptr(self.ox), self.nt,
                 self.C, self.H, self.W, self.bh, self.bw, ptr(out), stream())
        return out

    def gather_all(self, v):
        """All ranks' block corrections in tile order (identity on one rank)."""
        if self.ranks == 1:
            return v
        import torch.distributed as dist
        # NCCL gathers device tensors; other backends (the host-transport
        # harness, gloo) through host copies
        dev = v.device if dist.get_backend() == "nccl" else torch.device("cpu")
        pad = torch.zeros((self.chunk,) + tuple(v.shape[1:]), dtype=v.dtype, device=dev)
        pad[:self.nt] = v
        out = torch.empty((self.chunk * self.ranks,) + tuple(v.shape[1:]), dtype=v.dtype,
                          device=dev)
        dist.all_gather_into_tensor(out, pad)
        return out[:self.nt_all].to(v.device).contiguous()

    def scatter_add(self, g, v):
        """g += sum_b T(1/cover) * v_b (tonal.py:375-380); v holds all blocks."""
        if self.nt_all:
            call("sp_ras_scatter", dcode(g), ptr(g), ptr(v), ptr(self.tile_of), ptr(self.ys_t),
                 ptr(self.xs_t), ptr(self.rk0), ptr(self.rn), ptr(self.ck0), ptr(self.cn),
                 self.nbx, self.bh, self.bw, self.C, self.H, self.W, stream())
        return g

    # -- batched local products (cold solves to local_product_tol) ---------
    def _solve(self, bsym, active_h):
        self.solves += int(active_h.sum())
        u = torch.empty_like(bsym)
        call("sp_hier_solve_tiles", self.hier._h, ptr(bsym), ptr(u), 0, float(self.tol),
             int(self.inner_cycles), 100, ptr(active_h), ptr(self._iters), ptr(self._conv),
             stream())
        return u

    def apply_B(self, p, active_h, active_d):
        bsym = torch.empty_like(p)
        call("sp_masked_sym_rhs_tiles", dcode(p), ptr(p), ptr(self.tmask), ptr(bsym), self.C,
             self.bh, self.bw, self.nt, ptr(active_d), stream())
        return self._solve(bsym, active_h)

    def apply_Bt(self, y, active_h, active_d):
        w = self._solve(y, active_h)
        out = torch.empty_like(w)
        call("sp_ct_apply_tiles", dcode(w), ptr(w), ptr(self.tmask), ptr(out), self.C, self.bh,
             self.bw, self.nt, ptr(active_d), stream())
        return out

    def plane_dot(self, x, y, active_d):
        out = torch.zeros(self.nt * self.C, dtype=torch.float64, device=x.device)
        call("sp_plane_dot", dcode(x), ptr(x), ptr(y), self.bh * self.bw, self.nt * self.C,
             self.C, ptr(active_d), ptr(out), stream())
        return out.view(self.nt, self.C)

    def axpy(self, yout, x, z, coef, sign, active_d):
        coef_c = coef.contiguous()
        call("sp_plane_axpy", dcode(x), ptr(yout), ptr(x), ptr(z), ptr(coef_c), float(sign),
             self.bh * self.bw, self.nt * self.C, self.C, ptr(active_d), stream())

    def normal_cg(self, rhs, cap, tol):
        """tonal.py:267-294 for every tile at once (per-tile stopping)."""
        nt, C = self.nt, self.C
        v = torch.zeros_like(rhs)
        if nt == 0:
            return v
        dev = rhs.device
        r = rhs.clone()
        p = r.clone()
        ones = torch.ones(nt, dtype=torch.int32, device=dev)
        rs = self.plane_dot(r, r, ones)
        rs0 = rs.sum(1)
        active = rs0 != 0                                   # rs0 == 0 -> v = 0
        active &= rs.sum(1) > tol * rs0
        it = 0
        while it < cap:
            act_h = active.to(torch.int32).cpu().numpy()
            if not act_h.any():
                break
            act_d = torch.from_numpy(act_h).to(dev)
            bp = self.apply_B(p, act_h, act_d)
            mp = self.apply_Bt(bp, act_h, act_d)
            pmp = self.plane_dot(p, mp, act_d)
            alpha = torch.where(pmp > 0, rs / torch.where(pmp > 0, pmp, torch.ones_like(pmp)),
                                torch.zeros_like(pmp))
            anypos = (alpha > 0).any(1)
            active = active & anypos                        # break: no alpha > 0
            act_d = active.to(torch.int32)
            coef = alpha.reshape(-1)
            self.axpy(v, v, p, coef, +1.0, act_d)
            self.axpy(r, r, mp, coef, -1.0, act_d)
            rs_new = self.plane_dot(r, r, act_d)
            beta = torch.where(rs > 0, rs_new / torch.where(rs > 0, rs, torch.ones_like(rs)),
                               torch.zeros_like(rs))
            self.axpy(p, r, p, beta.reshape(-1), +1.0, act_d)
            rs = torch.where(active[:, None], rs_new, rs)
            it += 1
            active = active & (rs.sum(1) > tol * rs0)
        return v


def ras_tonal(f: Image, mask: Mask, init: TonalState | None = None,
              cfg: RasTonalConfig | None = None,
              solver: InpaintSolver | None = None) -> TonalState:
    """tonal.py:309-386: restricted additive Schwarz on the stored-value
    normal equations with averaging weights 1/cover."""
    if cfg is None:
        cfg = RasTonalConfig()
    if solver is None:
        solver = InpaintSolver()
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    m_t = mask.tensor()
    dt = solver.cfg.torch_dtype
    f64 = f.tensor(torch.float64)
    f_arr = f64.to(dt)
    C = f_arr.shape[0]
    sys_ = _TonalSystem(m_t, solver, C, cfg.inner_cycles, inner_tol=cfg.inner_tol,
                        cold_tol=cfg.cold_tol)
    if init is None:
        g = _where_mask(f_arr, m_t)
        u_warm = None
    else:
        g = _where_mask(init.g.tensor(dt), m_t)
        u_warm = init.u.tensor(dt)
    w_warm = None
    blocks = _RasBlocks(m_t, solver, C, cfg)
    t0 = time.perf_counter()
    history = []
    best_g = g.clone()
    best_mse = math.inf
    prev_mse = None
    outer = 0
    while outer < cfg.max_outer:
        u = sys_.apply_B(g, warm=u_warm)
        u_warm = u
        mse = mse_t(f_arr, u)
        history.append((outer, mse, time.perf_counter() - t0, sys_.solves))
        if mse < best_mse:
            best_mse, best_g = mse, g.clone()
        if prev_mse is not None and prev_mse - mse < cfg.rel_improvement * prev_mse:
            break
        prev_mse = mse
        rhs, w_warm = sys_.apply_Bt(f_arr - u, warm=w_warm)
        v = blocks.normal_cg(blocks.gather(rhs), cfg.local_iters, cfg.local_tol)
        g = blocks.scatter_add(g.clone(), blocks.gather_all(v))
        outer += 1
    total_inner = sys_.solves + blocks.solves
    state = _final_state(f64, m_t, sys_, best_g, u_warm, history, outer, cfg.final_tol)
    state.inner_solves = total_inner
    return state


# ---------------------------------------------------------------------------
# Voronoi / Richardson initialization
# ---------------------------------------------------------------------------

class _CellIndex:
    def __init__(self, lab_t, m):
        H, W = lab_t.shape
        dev = lab_t.device
        self.m = m
        self.perm = torch.empty(H * W, dtype=torch.int32, device=dev)
        self.start = torch.empty(m, dtype=torch.int32, device=dev)
        self.end = torch.empty(m, dtype=torch.int32, device=dev)
        call("sp_cell_index", ptr(lab_t), H, W, m, ptr(self.perm), ptr(self.start),
             ptr(self.end), stream())


def _cell_index(lab_t, m):
    return _CellIndex(lab_t.to(torch.int32).contiguous(), int(m))


def _voronoi_weights_t(lab_t, seeds_t, idx: _CellIndex, scheme="inverse-log"):
    """geometry.py:247-264 on the device -> (H, W) float64."""
    if scheme == "constant":
        code = 0
    elif scheme in ("inverse-log", "inverse-log-distance"):
        code = 1
    else:
        raise ValueError("scheme must be 'constant' or 'inverse-log'")
    lab_t = lab_t.to(torch.int32).contiguous()
    H, W = lab_t.shape
    sy = seeds_t[:, 0].to(torch.int32).contiguous()
    sx = seeds_t[:, 1].to(torch.int32).contiguous()
    w = torch.empty((H, W), dtype=torch.float64, device=lab_t.device)
    call("sp_vi_weights", ptr(lab_t), ptr(sy), ptr(sx), ptr(idx.perm), ptr(idx.start),
         ptr(idx.end), H, W, idx.m, code, ptr(w), stream())
    return w


def _cell_sum(idx: _CellIndex, vals):
    out = torch.empty(idx.m, dtype=torch.float64, device=vals.device)
    vals_c = vals.to(torch.float64).contiguous()
    call("sp_cell_sum", ptr(idx.perm), ptr(idx.start), ptr(idx.end), ptr(vals_c), idx.m,
         ptr(out), stream())
    return out


def voronoi_richardson_init(f: Image, mask: Mask, cfg: InitConfig | None = None,
                            solver: InpaintSolver | None = None,
                            labels: VoronoiLabels | None = None,
                            weights=None) -> TonalState:
    """tonal.py:417-476: damped cell-wise error balancing with one warm B
    product per step; stops at the first MSE increase, returns the best."""
    if cfg is None:
        cfg = InitConfig()
    if solver is None:
        solver = InpaintSolver()
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    m_t = mask.tensor()
    H, W = m_t.shape
    if labels is None:
        ws = workspace(H, W)
        ws.voronoi(m_t, None)
        lab_t = ws.labels_tensor()
        seeds_t = ws.seeds_tensor()
    else:
        lab_t = _lib.to_dev(np.asarray(labels.labels, np.int32))
        seeds_t = _lib.to_dev(np.asarray(labels.seeds, np.int32))
    m = int(seeds_t.shape[0])
    idx = _cell_index(lab_t, m)
    if weights is None:
        w = _voronoi_weights_t(lab_t, seeds_t, idx, cfg.weight_scheme)
    else:
        w = _lib.to_dev(np.asarray(weights, np.float64))
    dt = solver.cfg.torch_dtype
    f64 = f.tensor(torch.float64)
    f_arr = f64.to(dt).contiguous()
    C = f_arr.shape[0]
    sys_ = _TonalSystem(m_t, solver, C, cfg.inner_cycles, inner_tol=cfg.inner_tol)
    g = _where_mask(f_arr, m_t)
    sy = seeds_t[:, 0].to(torch.int32).contiguous()
    sx = seeds_t[:, 1].to(torch.int32).contiguous()
    t0 = time.perf_counter()
    u, _ = solver.inpaint(Image(f_arr), Mask(m_t))
    u = u.tensor(dt).contiguous()
    mse = mse_t(f_arr, u)
    history = [(0, mse, time.perf_counter() - t0, sys_.solves)]
    best_g, best_mse, prev_mse = g.clone(), mse, mse
    steps = 0
    for k in range(1, cfg.max_steps + 1):
        call("sp_vi_step", dcode(g), ptr(idx.perm), ptr(idx.start), ptr(idx.end), ptr(w),
             ptr(f_arr), ptr(u), ptr(sy), ptr(sx), m, C, H, W, float(cfg.tau), ptr(g),
             stream())
        u = sys_.apply_B(g, warm=u)
        mse = mse_t(f_arr, u)
        steps = k
        history.append((k, mse, time.perf_counter() - t0, sys_.solves))
        if mse < best_mse:
            best_mse, best_g = mse, g.clone()
        if cfg.stop_on_mse_increase and mse > prev_mse:
            break
        prev_mse = mse
    return _final_state(f64, m_t, sys_, best_g, u, history, steps, cfg.final_tol)


def neighbor_balance_init(f: Image, u: Image, mask: Mask, solver: InpaintSolver | None = None,
                          final_tol: float = 1e-6) -> TonalState:
    """tonal.py:389-414: 3x3 (border-clipped) mean signed error added to the
    stored values, one CUDA pass (sp_neighbor_balance, scipy `correlate`
    summation order, bit-exact)."""
    f64 = f.tensor(torch.float64)
    u_t = u.tensor()
    if u_t.dtype not in (torch.float32, torch.float64):
        u_t = u_t.to(torch.float64)
    m_t = mask.tensor()
    C, H, W = u_t.shape
    if tuple(f64.shape) != (C, H, W) or tuple(m_t.shape) != (H, W):
        raise ValueError("image, reconstruction and mask dimensions disagree")
    g = torch.empty_like(u_t)
    call("sp_neighbor_balance", dcode(u_t), ptr(f64), ptr(u_t), ptr(m_t), ptr(g), C, H, W,
         stream())
    if solver is None:
        unew = u.copy()
        return TonalState(g=Image(g), u=unew, mse=mse_t(f64, unew.tensor()))
    sys_ = _TonalSystem(m_t, solver, g.shape[0])
    return _final_state(f64, m_t, sys_, g.to(sys_.dtype), u_t.to(sys_.dtype), [], 1, final_tol)


def dense_tonal_oracle(f: Image, mask: Mask, max_pixels: int = 4096) -> TonalState:
    """tonal.py:479-507: dense verification oracle (desk scale only; dense
    linear algebra through torch on the device)."""
    n = f.height * f.width
    if n > max_pixels:
        raise ValueError(f"dense oracle limited to {max_pixels} pixels")
    if mask.count == 0:
        raise ValueError("singular system: empty mask")
    dev = _lib.device()
    m = torch.as_tensor(np.asarray(mask.indicator), device=dev).reshape(-1).bool()
    h, w = f.height, f.width
    eye = torch.eye(n, dtype=torch.float64, device=dev)
    # A = C + (I - C) L, assembled from the 5-point stencil
    idx = torch.arange(n, device=dev)
    yy, xx = idx // w, idx % w
    L = torch.zeros((n, n), dtype=torch.float64, device=dev)
    for dy, dx in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ny, nx = yy + dy, xx + dx
        ok = (ny >= 0) & (ny < h) & (nx >= 0) & (nx < w)
        L[idx[ok], idx[ok]] += 1.0
        L[idx[ok], (ny * w + nx)[ok]] -= 1.0
    A = torch.where(m[:, None], eye, L)
    midx = torch.nonzero(m).reshape(-1)
    rhs = torch.zeros((n, midx.numel()), dtype=torch.float64, device=dev)
    rhs[midx, torch.arange(midx.numel(), device=dev)] = 1.0
    Bc = torch.linalg.solve(A, rhs)
    normal = Bc.T @ Bc
    fd = f.tensor(torch.float64)
    g = torch.zeros_like(fd)
    u = torch.zeros_like(fd)
    for ch in range(fd.shape[0]):
        gk = torch.linalg.solve(normal, Bc.T @ fd[ch].reshape(-1))
        g[ch].view(-1)[midx] = gk
        u[ch] = (Bc @ gk).view(h, w)
    return TonalState(g=Image(g), u=Image(u), mse=mse_t(fd, u))
