"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference data-optimization path (`sparsepaint` 0.1.0,
/root/reference/pkg/src/sparsepaint) in numpy + the C kernel table in
``sp_oracle.c``.  It is the checker for the CUDA product
(``paper_2401_06747_b200``) and the timed CPU baseline of ``bench.py``.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import it; the product never does.

Parity pinning: tests/test_oracle_golden.py checks every function here
against fixtures that tests/golden/make_golden.py produced by running the
reference itself (numba backend) in the build container.  Third-party
arithmetic used by the reference and restated here: numpy PCG64 +
``Generator.random`` / ``choice`` (used directly), numpy ``sum`` /
``lexsort`` / ``unique`` / ``bincount`` (used directly), scipy
``ndimage.gaussian_filter`` (used directly).

Arrays: images are (C, H, W) float32/float64, masks (H, W) uint8.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libsp_oracle.so")
_lib = None


def build(force=False):
    """Compile sp_oracle.c (gcc, OpenMP, no FMA contraction)."""
    src = os.path.join(_HERE, "sp_oracle.c")
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= os.path.getmtime(src)):
        return _SO
    os.makedirs(os.path.dirname(_SO), exist_ok=True)
    tmp = _SO + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off",
                           "-fPIC", "-shared", "-o", tmp, src, "-lm"])
    os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _sfx(a):
    if a.dtype == np.float32:
        return "f32"
    if a.dtype == np.float64:
        return "f64"
    raise TypeError(f"unsupported dtype {a.dtype}")


def _c(a, dtype=None):
    return np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))


# ---------------------------------------------------------------------------
# kernel table (kernels/__init__.py:12-29, numba_impl.py)
# ---------------------------------------------------------------------------

def negated_laplacian(x, inv_h2):
    x = _c(x)
    out = np.empty_like(x)
    getattr(lib(), "ora_negated_laplacian_" + _sfx(x))(
        _p(x), _p(out), *map(ctypes.c_int, x.shape), ctypes.c_double(inv_h2))
    return out


def _masked(name, x, mask, inv_h2):
    x = _c(x)
    mask = _c(mask, np.uint8)
    out = np.empty_like(x)
    getattr(lib(), f"ora_{name}_" + _sfx(x))(
        _p(x), _p(mask), _p(out), *map(ctypes.c_int, x.shape),
        ctypes.c_double(inv_h2))
    return out


def inpaint_matvec(x, mask, inv_h2):
    return _masked("inpaint_matvec", x, mask, inv_h2)


def sym_matvec(x, mask, inv_h2):
    return _masked("sym_matvec", x, mask, inv_h2)


def sym_rhs(b, mask, inv_h2):
    return _masked("sym_rhs", b, mask, inv_h2)


def ct_apply(w, mask, inv_h2):
    return _masked("ct_apply", w, mask, inv_h2)


def sym_residual(u, bsym, mask, inv_h2):
    u = _c(u)
    bsym = _c(bsym, u.dtype)
    mask = _c(mask, np.uint8)
    r = np.empty_like(u)
    norms = np.zeros(u.shape[0], np.float64)
    getattr(lib(), "ora_sym_residual_" + _sfx(u))(
        _p(u), _p(bsym), _p(mask), _p(r), _p(norms), *map(ctypes.c_int, u.shape),
        ctypes.c_double(inv_h2))
    return r, norms


def oras_apply(u, r, mask, xs, ys, bh, bw, gamma, taus, cap, weights, inv_h2):
    """Mutates ``u`` (numba_impl.py:161-263)."""
    assert u.flags.c_contiguous
    r = _c(r, u.dtype)
    mask = _c(mask, np.uint8)
    xs = _c(xs, np.int64)
    ys = _c(ys, np.int64)
    taus = _c(taus, np.float64)
    weights = _c(weights, u.dtype)
    getattr(lib(), "ora_oras_apply_" + _sfx(u))(
        _p(u), _p(r), _p(mask), _p(xs), ctypes.c_int(xs.size), _p(ys),
        ctypes.c_int(ys.size), ctypes.c_int(bh), ctypes.c_int(bw),
        ctypes.c_double(gamma), _p(taus), ctypes.c_long(cap), _p(weights),
        ctypes.c_double(inv_h2), *map(ctypes.c_int, u.shape))


def restrict_values(fine):
    fine = _c(fine)
    c, h, w = fine.shape
    out = np.zeros((c, (h + 1) // 2, (w + 1) // 2), fine.dtype)
    getattr(lib(), "ora_restrict_values_" + _sfx(fine))(
        _p(fine), _p(out), ctypes.c_int(c), ctypes.c_int(h), ctypes.c_int(w))
    return out


def restrict_mask(mask, values):
    mask = _c(mask, np.uint8)
    values = _c(values)
    c = values.shape[0]
    h, w = mask.shape
    cm = np.zeros(((h + 1) // 2, (w + 1) // 2), np.uint8)
    cv = np.zeros((c,) + cm.shape, values.dtype)
    getattr(lib(), "ora_restrict_mask_" + _sfx(values))(
        _p(mask), _p(values), _p(cm), _p(cv), ctypes.c_int(c), ctypes.c_int(h),
        ctypes.c_int(w))
    return cm, cv


def prolongate(coarse, h, w):
    coarse = _c(coarse)
    c, ch, cw = coarse.shape
    out = np.empty((c, h, w), coarse.dtype)
    getattr(lib(), "ora_prolongate_" + _sfx(coarse))(
        _p(coarse), _p(out), ctypes.c_int(c), ctypes.c_int(ch), ctypes.c_int(cw),
        ctypes.c_int(h), ctypes.c_int(w))
    return out


def jfa_run(labels, seeds, steps):
    labels = _c(labels, np.int32)
    seeds = _c(seeds, np.int64)
    steps = _c(steps, np.int64)
    out = np.empty_like(labels)
    h, w = labels.shape
    lib().ora_jfa_run(_p(labels), _p(out), _p(seeds), ctypes.c_long(seeds.shape[0]),
                      _p(steps), ctypes.c_int(steps.size), ctypes.c_int(h),
                      ctypes.c_int(w))
    return out


def jfa_dist2(labels, seeds):
    labels = _c(labels, np.int32)
    seeds = _c(seeds, np.int64)
    out = np.empty(labels.shape, np.int64)
    lib().ora_jfa_dist2(_p(labels), _p(seeds), ctypes.c_long(seeds.shape[0]), _p(out),
                        *map(ctypes.c_int, labels.shape))
    return out


def fs_dither(dens):
    dens = _c(dens, np.float64)
    out = np.empty(dens.shape, np.uint8)
    lib().ora_fs_dither(_p(dens), _p(out), *map(ctypes.c_int, dens.shape))
    return out


def assign_triangles(tris, vy, vx, h, w):
    tris = _c(tris, np.int64).reshape(-1, 3)
    vy = _c(vy, np.int64)
    vx = _c(vx, np.int64)
    out = np.empty((h, w), np.int32)
    lib().ora_assign_triangles(_p(tris), ctypes.c_long(tris.shape[0]), _p(vy),
                               _p(vx), ctypes.c_int(h), ctypes.c_int(w), _p(out))
    return out


def fallback_assign(assign, labels, seed_min_tri):
    assign = _c(assign, np.int32)
    labels = _c(labels, np.int32)
    smt = _c(seed_min_tri, np.int32)
    out = np.empty_like(assign)
    lib().ora_fallback_assign(_p(assign), _p(labels), _p(smt), _p(out),
                              *map(ctypes.c_int, assign.shape))
    return out


def reduce_cells(assign, err, ntris):
    assign = _c(assign, np.int32)
    err = _c(err, np.float64)
    sums = np.zeros(ntris, np.float64)
    ai = np.full(ntris, -1, np.int64)
    av = np.full(ntris, -1.0, np.float64)
    lib().ora_reduce_cells(_p(assign), _p(err), ctypes.c_long(ntris), _p(sums),
                           _p(ai), _p(av), *map(ctypes.c_int, assign.shape))
    return sums, ai, av


KERNEL_NAMES = ["negated_laplacian", "inpaint_matvec", "sym_matvec", "sym_rhs",
                "ct_apply", "sym_residual", "oras_apply", "restrict_values",
                "restrict_mask", "prolongate", "jfa_run", "jfa_dist2",
                "fs_dither", "assign_triangles", "fallback_assign",
                "reduce_cells"]


# ---------------------------------------------------------------------------
# block decomposition + multigrid (solver.py:134-590)
# ---------------------------------------------------------------------------

def starts(dim, size, stride):
    """solver.py:134-139."""
    if dim <= size:
        return np.array([0], np.int64)
    n = math.ceil((dim - size) / stride) + 1
    return np.array([min(i * stride, dim - size) for i in range(n)], np.int64)


_DECOMP = {}


def build_decomposition(h, w, block=32, overlap=6):
    """solver.py:142-197: ramp weights min(dist+1, overlap), pointwise
    normalized; the last covering block takes the exact complement."""
    key = (h, w, block, overlap)
    if key in _DECOMP:
        return _DECOMP[key]
    bh, bw = min(block, h), min(block, w)
    ys = starts(h, bh, block - overlap)
    xs = starts(w, bw, block - overlap)
    nbx = xs.size
    nb = ys.size * nbx
    ii = np.arange(bh, dtype=np.float64)[:, None]
    jj = np.arange(bw, dtype=np.float64)[None, :]
    raw = np.empty((nb, bh, bw))
    for bi in range(nb):
        y0, x0 = int(ys[bi // nbx]), int(xs[bi % nbx])
        di = np.full((bh, bw), float(max(h, w)))
        if y0 > 0:
            di = np.minimum(di, ii)
        if y0 + bh < h:
            di = np.minimum(di, bh - 1 - ii)
        if x0 > 0:
            di = np.minimum(di, jj)
        if x0 + bw < w:
            di = np.minimum(di, bw - 1 - jj)
        raw[bi] = np.minimum(di + 1.0, float(overlap))
    total = np.zeros((h, w))
    last = np.full((h, w), -1, np.int64)
    for bi in range(nb):
        y0, x0 = int(ys[bi // nbx]), int(xs[bi % nbx])
        total[y0:y0 + bh, x0:x0 + bw] += raw[bi]
        last[y0:y0 + bh, x0:x0 + bw] = bi
    acc = np.zeros((h, w))
    wts = np.empty_like(raw)
    for bi in range(nb):
        y0, x0 = int(ys[bi // nbx]), int(xs[bi % nbx])
        sl = (slice(y0, y0 + bh), slice(x0, x0 + bw))
        wn = np.where(last[sl] == bi, 1.0 - acc[sl], raw[bi] / total[sl])
        acc[sl] += wn
        wts[bi] = wn
    d = dict(bh=bh, bw=bw, ys=ys, xs=xs, weights=wts, nb=nb)
    _DECOMP[key] = d
    return d


class Report:
    def __init__(self):
        self.iterations = 0
        self.residuals = []
        self.converged = False
        self.seconds = 0.0


class Hierarchy:
    """GridHierarchy (solver.py:221-590) restated on raw arrays."""

    def __init__(self, mask, values, dtype=np.float32, block=32, overlap=6,
                 levels=0, pre=1, post=1, cycles=1, alpha=1.0, rho=0.25,
                 max_cycles=100):
        self.dtype = np.dtype(dtype)
        self.block, self.overlap, self.rho = block, overlap, rho
        self.pre, self.post, self.cycles = pre, post, cycles
        self.max_cycles = max_cycles
        self.gamma = (1.0 - alpha) / (1.0 + alpha)
        m = np.ascontiguousarray(mask, np.uint8)
        v = None if values is None else values.astype(self.dtype)
        self.masks, self.values, self.decomps = [], [], []
        lv = 0
        while True:
            h, w = m.shape
            self.masks.append(m)
            self.values.append(v)
            self.decomps.append(build_decomposition(h, w, block, overlap))
            lv += 1
            if levels > 0:
                if lv >= levels or max(h, w) <= 2:
                    break
            elif max(h, w) <= block:
                break
            if v is None:
                m, _ = restrict_mask(m, np.zeros((1, h, w), self.dtype))
            else:
                m, v = restrict_mask(m, v)
        self.nlevels = len(self.masks)

    def residual(self, lv, u, bsym):
        return sym_residual(u, bsym, self.masks[lv], 1.0)

    def smooth(self, lv, u, bsym, sweeps):
        d = self.decomps[lv]
        n = self.masks[lv].size
        wts = d["weights"].astype(u.dtype)
        for _ in range(sweeps):
            r, norms = self.residual(lv, u, bsym)
            taus = self.rho * (d["bh"] * d["bw"] / n) * norms
            oras_apply(u, r, self.masks[lv], d["xs"], d["ys"], d["bh"], d["bw"],
                       self.gamma, taus, d["bh"] * d["bw"], wts, 1.0)
        return u

    def enforce(self, lv, u, bsym):
        m = self.masks[lv].astype(bool)
        for ch in range(u.shape[0]):
            u[ch][m] = bsym[ch][m]
        return u

    def vcycle(self, lv, u, bsym):
        if lv == self.nlevels - 1:
            return self.smooth(lv, u, bsym, self.pre + self.post)
        self.smooth(lv, u, bsym, self.pre)
        r, _ = self.residual(lv, u, bsym)
        bc = sym_rhs(restrict_values(r), self.masks[lv + 1], 1.0)
        e = np.zeros_like(bc)
        self.enforce(lv + 1, e, bc)
        self.vcycle(lv + 1, e, bc)
        h, w = self.masks[lv].shape
        u += prolongate(e, h, w)
        self.enforce(lv, u, bsym)
        self.smooth(lv, u, bsym, self.post)
        return u

    def level_rhs(self, lv, dtype):
        m = self.masks[lv]
        b = np.where(m[None].astype(bool), self.values[lv], 0).astype(dtype)
        return sym_rhs(b, m, 1.0)

    def cascade(self, channels, dtype):
        lv = self.nlevels - 1
        u = np.zeros((channels,) + self.masks[lv].shape, dtype)
        b = self.level_rhs(lv, dtype)
        self.enforce(lv, u, b)
        self.smooth(lv, u, b, 1)
        for lv in range(self.nlevels - 2, -1, -1):
            h, w = self.masks[lv].shape
            u = prolongate(u, h, w)
            b = self.level_rhs(lv, dtype)
            self.enforce(lv, u, b)
            self.smooth(lv, u, b, 1)
        return u

    def solve_sym(self, bsym, init=None, tol=None, cycles=None, max_cycles=None,
                  cascade=False):
        """solver.py:328-372."""
        t0 = time.perf_counter()
        rep = Report()
        bsym = np.ascontiguousarray(bsym)
        if init is not None:
            u = np.ascontiguousarray(init.astype(bsym.dtype, copy=True))
        elif cascade and self.nlevels > 1:
            u = self.cascade(bsym.shape[0], bsym.dtype)
        else:
            u = np.zeros_like(bsym)
        self.enforce(0, u, bsym)
        if tol is None:
            n = self.cycles if cycles is None else cycles
            for _ in range(n):
                self.vcycle(0, u, bsym)
            rep.iterations = n
            rep.converged = True
        else:
            cap = self.max_cycles if max_cycles is None else max_cycles
            bd = bsym.ravel().astype(np.float64)
            bnorm = math.sqrt(float(np.dot(bd, bd)))
            scale = bnorm if bnorm > 0 else 1.0
            done = 0
            while True:
                _, norms = self.residual(0, u, bsym)
                rel = math.sqrt(float(norms.sum())) / scale
                rep.residuals.append(rel)
                if rel <= tol:
                    rep.converged = True
                    break
                if done >= cap:
                    break
                self.vcycle(0, u, bsym)
                done += 1
            rep.iterations = done
        rep.seconds = time.perf_counter() - t0
        return u, rep


class SolverCfg:
    """MultigridConfig defaults (solver.py:49-82)."""

    def __init__(self, dtype="float32", tol=1e-4, cycles=1, max_cycles=100,
                 mode="fmg", levels=0, pre=1, post=1, block=32, overlap=6,
                 alpha=1.0, rho=0.25):
        self.dtype = np.dtype(dtype)
        self.tol, self.cycles, self.max_cycles = tol, cycles, max_cycles
        self.mode, self.levels, self.pre, self.post = mode, levels, pre, post
        self.block, self.overlap, self.alpha, self.rho = block, overlap, alpha, rho

    def hierarchy(self, mask, values):
        return Hierarchy(mask, values, self.dtype, self.block, self.overlap,
                         self.levels, self.pre, self.post, self.cycles,
                         self.alpha, self.rho, self.max_cycles)


def inpaint(f, mask, cfg=None, init=None, tol="cfg"):
    """solver.py:485-511: returns (u, report); u[mask] = f[mask] exactly."""
    cfg = cfg or SolverCfg()
    mask = np.ascontiguousarray(mask, np.uint8)
    if not mask.any():
        raise ValueError("singular system: empty mask")
    f_arr = np.ascontiguousarray(f, cfg.dtype)
    hier = cfg.hierarchy(mask, f_arr)
    b = np.where(mask[None].astype(bool), f_arr, 0)
    bsym = sym_rhs(b, mask, 1.0)
    init_arr = None if init is None else init.astype(cfg.dtype)
    u, rep = hier.solve_sym(bsym, init=init_arr,
                            tol=cfg.tol if tol == "cfg" else tol,
                            cycles=cfg.cycles, max_cycles=cfg.max_cycles,
                            cascade=(cfg.mode == "fmg" and init is None))
    m = mask.astype(bool)
    for ch in range(u.shape[0]):
        u[ch][m] = f_arr[ch][m]
    return u, rep


# ---------------------------------------------------------------------------
# geometry (geometry.py:76-272)
# ---------------------------------------------------------------------------

def steps_for(max_dim, start_hint):
    """geometry.py:76-89: [1] + halving from start."""
    if start_hint is not None and start_hint >= 1:
        start = 1 << max(0, math.ceil(math.log2(max(1.0, start_hint))))
        start = min(start, max(1, max_dim // 2))
    elif max_dim >= 2:
        start = 1 << (math.ceil(math.log2(max_dim)) - 1)
    else:
        start = 1
    out = [1]
    while start >= 1:
        out.append(start)
        start //= 2
    return np.array(out, np.int64)


def jump_flood_voronoi(mask, start_hint=None):
    """geometry.py:92-110 -> (labels i32, seeds i64 (m,2), max_radius)."""
    ys, xs = np.nonzero(mask)
    if ys.size == 0:
        raise ValueError("mask has no stored pixels to seed from")
    seeds = np.stack([ys, xs], axis=1).astype(np.int64)
    h, w = mask.shape
    lab = np.full((h, w), -1, np.int32)
    lab[ys, xs] = np.arange(ys.size, dtype=np.int32)
    lab = jfa_run(lab, seeds, steps_for(max(h, w), start_hint))
    d2 = jfa_dist2(lab, seeds)
    return lab, seeds, float(math.sqrt(float(d2.max())))


def delaunay_from_voronoi(lab, m):
    """geometry.py:113-185 -> (triangles i32 (T,3), edges i32 (E,2))."""
    h, w = lab.shape
    pairs = []
    for a, b in ((lab[:, :-1].ravel(), lab[:, 1:].ravel()),
                 (lab[:-1, :].ravel(), lab[1:, :].ravel())):
        k = a != b
        pairs.append(np.stack([np.minimum(a[k], b[k]), np.maximum(a[k], b[k])], 1))
    allp = np.concatenate(pairs, 0)
    edges = np.unique(allp, axis=0) if allp.size else np.zeros((0, 2), np.int64)
    parts = []
    if h >= 2 and w >= 2 and m >= 3:
        tl, tr = lab[:-1, :-1].ravel(), lab[:-1, 1:].ravel()
        bl, br = lab[1:, :-1].ravel(), lab[1:, 1:].ravel()
        srt = np.sort(np.stack([tl, tr, bl, br], 1), 1)
        dup = srt[:, 1:] == srt[:, :-1]
        nd = 4 - dup.sum(1)
        k3 = nd == 3
        if k3.any():
            s, d = srt[k3], dup[k3]
            parts.append(np.stack([s[:, 0], np.where(d[:, 0], s[:, 2], s[:, 1]),
                                   np.where(d[:, 2], s[:, 2], s[:, 3])], 1))
        k4 = nd == 4
        if k4.any():
            a, b, c, d = tl[k4], tr[k4], bl[k4], br[k4]
            d1lo, d1hi = np.minimum(a, d), np.maximum(a, d)
            d2lo, d2hi = np.minimum(b, c), np.maximum(b, c)
            use1 = ((d1lo < d2lo) | ((d1lo == d2lo) & (d1hi <= d2hi)))[:, None]
            ta = np.where(use1, np.stack([a, b, d], 1), np.stack([a, b, c], 1))
            tb = np.where(use1, np.stack([a, c, d], 1), np.stack([b, c, d], 1))
            parts += [np.sort(ta, 1), np.sort(tb, 1)]
    tris = (np.unique(np.concatenate(parts, 0), axis=0).astype(np.int32)
            if parts else np.zeros((0, 3), np.int32))
    return tris, edges.astype(np.int32)


def seed_min_triangle(tris, m):
    """geometry.py:188-194: lowest triangle index incident to each seed."""
    out = np.full(m, -1, np.int32)
    if tris.shape[0]:
        t = np.repeat(np.arange(tris.shape[0], dtype=np.int32), 3)
        v = tris.ravel().astype(np.int64)
        np.minimum.at(out.view(np.uint32), v, t.view(np.uint32))
    return out


def accumulate_errors(tris, err, lab, seeds):
    """geometry.py:197-223 -> (sums f64, amax i64, amax_val f64, unassigned)."""
    err = np.asarray(err, np.float64)
    if tris.shape[0] == 0:
        return np.zeros(0), np.zeros(0, np.int64), np.zeros(0), float(err.sum())
    h, w = err.shape
    assign = assign_triangles(tris.astype(np.int64), seeds[:, 0], seeds[:, 1], h, w)
    smt = seed_min_triangle(tris, seeds.shape[0])
    assign = fallback_assign(assign, lab, smt)
    s, ai, av = reduce_cells(assign, err, tris.shape[0])
    return s, ai, av, 0.0


def voronoi_cell_errors(lab, m, err):
    """geometry.py:226-244."""
    fl = lab.ravel().astype(np.int64)
    fe = np.asarray(err, np.float64).ravel()
    sums = np.bincount(fl, weights=fe, minlength=m)
    order = np.lexsort((np.arange(fl.size), -fe, fl))
    first = np.ones(order.size, bool)
    first[1:] = fl[order[1:]] != fl[order[:-1]]
    ai = np.full(m, -1, np.int64)
    av = np.full(m, -1.0)
    lead = order[first]
    ai[fl[lead]] = lead
    av[fl[lead]] = fe[lead]
    return sums, ai, av


def voronoi_weights(lab, seeds, scheme="inverse-log"):
    """geometry.py:247-264."""
    fl = lab.ravel().astype(np.int64)
    m = seeds.shape[0]
    if scheme == "constant":
        raw = np.ones(fl.size)
    elif scheme in ("inverse-log", "inverse-log-distance"):
        d2 = jfa_dist2(lab, seeds)
        raw = 1.0 / np.log(2.0 + np.sqrt(d2.ravel().astype(np.float64)))
    else:
        raise ValueError("scheme must be 'constant' or 'inverse-log'")
    tot = np.bincount(fl, weights=raw, minlength=m)
    return (raw / tot[fl]).reshape(lab.shape)


def cell_weighted_average(lab, m, weights, plane):
    """geometry.py:267-272."""
    return np.bincount(lab.ravel().astype(np.int64),
                       weights=(weights * plane).ravel(), minlength=m)


# ---------------------------------------------------------------------------
# spatial optimization (spatial.py:71-277)
# ---------------------------------------------------------------------------

def target_count(density, n):
    t = int(math.floor(density * n))
    if t < 1:
        raise ValueError("density too low: no pixel budget")
    return t


def schedule(total, iterations, growth=1.0, initial_fraction=None):
    """spatial.py:151-181."""
    wts = [growth ** i for i in range(iterations + 1)]
    if initial_fraction is None:
        init = int(round(total * wts[0] / sum(wts)))
    else:
        init = int(math.floor(initial_fraction * total))
    init = max(1, min(total, init))
    rem = total - init
    counts = [0] * iterations
    if rem > 0:
        def seq(m1):
            out, m = [], m1
            for _ in range(iterations):
                out.append(m)
                m = int(round(growth * m))
            return out
        lo, hi = 0, rem
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if sum(seq(mid)) <= rem:
                lo = mid
            else:
                hi = mid - 1
        counts = seq(lo)
        counts[-1] += rem - sum(counts)
    return init, counts


def uniform_random_mask(h, w, count, seed=0):
    n = h * w
    if not 1 <= count <= n:
        raise ValueError("count out of range")
    picks = np.random.default_rng(seed).choice(n, size=count, replace=False)
    m = np.zeros(n, np.uint8)
    m[picks] = 1
    return m.reshape(h, w)


def exact_count(bits, dens, target):
    """spatial.py:90-104."""
    fb = bits.ravel().astype(bool).copy()
    fd = dens.ravel()
    cnt = int(fb.sum())
    idx = np.arange(fb.size)
    if cnt > target:
        cand = idx[fb]
        fb[cand[np.lexsort((cand, fd[cand]))[:cnt - target]]] = False
    elif cnt < target:
        cand = idx[~fb]
        fb[cand[np.lexsort((cand, -fd[cand]))[:target - cnt]]] = True
    return fb.reshape(bits.shape)


def laplacian_density_map(f, density, sigma=1.0):
    """spatial.py:107-120."""
    from scipy.ndimage import gaussian_filter
    data = np.asarray(f, np.float64)
    if sigma > 0:
        data = np.stack([gaussian_filter(c, sigma, mode="reflect") for c in data])
    mag = np.abs(negated_laplacian(data, 1.0)).sum(axis=0)
    total = mag.sum()
    if total == 0:
        return None
    return np.clip(mag * (density * mag.size / total), 0.0, 1.0)


def analytic_mask(f, density, dither="floyd-steinberg", sigma=1.0, seed=0,
                  count=None):
    """spatial.py:123-148."""
    f = np.asarray(f)
    _, h, w = f.shape
    n = h * w
    target = target_count(density, n) if count is None else int(count)
    if target < 1:
        raise ValueError("density too low: no pixel budget")
    if target >= n:
        return np.ones((h, w), np.uint8)
    dens = laplacian_density_map(f, target / n, sigma)
    if dens is None:
        return uniform_random_mask(h, w, target, seed)
    if dither == "floyd-steinberg":
        bits = fs_dither(dens).astype(bool)
    elif dither == "random":
        bits = np.random.default_rng(seed).random(dens.shape) < dens
    else:
        raise ValueError("dither must be 'floyd-steinberg' or 'random'")
    return exact_count(bits, dens, target).astype(np.uint8)


def error_map(u, f):
    d = u.astype(np.float64) - f.astype(np.float64)
    return (d * d).sum(axis=0)


def mse(a, b):
    d = a.astype(np.float64) - b.astype(np.float64)
    return float(np.mean(d * d))


def psnr(m):
    return math.inf if m == 0 else 10.0 * math.log10(255.0 ** 2 / m)


def select_picks(sums, amax, mask_flat, want):
    """spatial.py:251-259: highest sums first, index ties ascending."""
    order = np.lexsort((np.arange(sums.size), -sums))
    picked = []
    for t in order:
        if len(picked) >= want:
            break
        px = amax[t]
        if px < 0 or mask_flat[px]:
            continue
        picked.append(int(px))
    return picked


def fill_highest_error(mask, err, want):
    fe = err.ravel()
    idx = np.arange(fe.size)
    cand = idx[~mask.ravel().astype(bool)]
    out = mask.ravel().copy()
    out[cand[np.lexsort((cand, -fe[cand]))[:want]]] = 1
    return out.reshape(mask.shape)


def delaunay_densify(f, density=0.05, iterations=20, growth=1.0,
                     initial_fraction=None, initial_scheme="laplacian-dither",
                     init_sigma=1.0, seed=0, cfg=None, partition="delaunay",
                     trace=None):
    """spatial.py:200-277 -> (mask, u, history).  ``trace`` (a list) receives
    one dict per iteration for lockstep parity checks."""
    cfg = cfg or SolverCfg()
    f = np.asarray(f, np.float64) if np.asarray(f).dtype.kind != "f" else np.asarray(f)
    _, h, w = f.shape
    n = h * w
    total = target_count(density, n)
    init_count, counts = schedule(total, iterations, growth, initial_fraction)
    if initial_scheme == "laplacian-dither":
        mask = analytic_mask(f, init_count / n, dither="random", sigma=init_sigma,
                             seed=seed, count=init_count)
    else:
        mask = uniform_random_mask(h, w, init_count, seed)
    hist = []
    t0 = time.perf_counter()
    u = None
    hint = None
    carry = 0
    for it, quota in enumerate(counts):
        u, _ = inpaint(f, mask, cfg, init=u)
        err = error_map(u, f)
        m_ = mse(f, u)
        hist.append((it, int(mask.sum()), m_, psnr(m_), time.perf_counter() - t0))
        want = quota + carry
        if want <= 0:
            carry = 0
            continue
        lab, seeds, rad = jump_flood_voronoi(mask, hint)
        hint = rad
        if partition == "delaunay":
            tris, _ = delaunay_from_voronoi(lab, seeds.shape[0])
            sums, amax, _, _ = accumulate_errors(tris, err, lab, seeds)
        else:
            tris = None
            sums, amax, _ = voronoi_cell_errors(lab, seeds.shape[0], err)
        picked = select_picks(sums, amax, mask.ravel(), want)
        if trace is not None:
            trace.append(dict(mask=mask.copy(), err=err, labels=lab, tris=tris,
                              sums=sums, amax=amax, picked=np.array(picked, np.int64),
                              want=want))
        if picked:
            mask = mask.copy()
            mask.ravel()[np.array(picked, np.int64)] = 1
        carry = want - len(picked)
    if carry > 0:
        u, _ = inpaint(f, mask, cfg, init=u)
        mask = fill_highest_error(mask, error_map(u, f), carry)
    u, _ = inpaint(f, mask, cfg, init=u)
    m_ = mse(f, u)
    hist.append((len(counts), int(mask.sum()), m_, psnr(m_), time.perf_counter() - t0))
    assert int(mask.sum()) == total
    return mask, u, hist


# ---------------------------------------------------------------------------
# tonal optimization (tonal.py:86-476)
# ---------------------------------------------------------------------------

def chan_dot(a, b):
    return np.array([float(np.dot(a[c].ravel().astype(np.float64),
                                  b[c].ravel().astype(np.float64)))
                     for c in range(a.shape[0])])


class TonalSystem:
    """tonal.py:100-144."""

    def __init__(self, mask, cfg, inner_cycles=1, inner_tol=None, cold_tol=1e-4,
                 cold_max_cycles=100):
        self.mask = np.ascontiguousarray(mask, np.uint8)
        self.hier = cfg.hierarchy(self.mask, None)
        self.inner_cycles, self.inner_tol = inner_cycles, inner_tol
        self.cold_tol, self.cold_max_cycles = cold_tol, cold_max_cycles
        self.dtype = cfg.dtype
        self.solves = 0

    def solve(self, bsym, warm, tol=None, cycles=None):
        self.solves += 1
        if tol is None:
            if self.inner_tol is not None:
                tol = self.inner_tol
            elif warm is None:
                tol = self.cold_tol
        u, _ = self.hier.solve_sym(bsym, init=warm, tol=tol,
                                   cycles=self.inner_cycles if cycles is None else cycles,
                                   max_cycles=self.cold_max_cycles)
        return u

    def apply_B(self, x, warm=None, tol=None, cycles=None):
        b = np.where(self.mask[None].astype(bool), x, 0).astype(self.dtype)
        return self.solve(sym_rhs(b, self.mask, 1.0), warm, tol, cycles)

    def apply_Bt(self, y, warm=None, tol=None, cycles=None):
        w = self.solve(y.astype(self.dtype), warm, tol, cycles)
        return ct_apply(w, self.mask, 1.0), w


def final_state(f, mask, sys_, g_best, warm, history, iterations, final_tol):
    """tonal.py:183-195 -> dict(g, u, mse, ...)."""
    b = np.where(sys_.mask[None].astype(bool), g_best, 0).astype(sys_.dtype)
    u, rep = sys_.hier.solve_sym(sym_rhs(b, sys_.mask, 1.0), init=warm, tol=final_tol)
    sys_.solves += 1
    m = mask.astype(bool)
    for ch in range(u.shape[0]):
        u[ch][m] = g_best[ch][m]
    return dict(g=g_best.copy(), u=u, mse=mse(f, u), history=history,
                iterations=iterations, inner_solves=sys_.solves,
                converged=rep.converged)


def voronoi_richardson_init(f, mask, cfg=None, tau=1.0, weight_scheme="inverse-log",
                            max_steps=20, stop_on_mse_increase=True, inner_cycles=2,
                            inner_tol=None, final_tol=1e-6):
    """tonal.py:417-476."""
    cfg = cfg or SolverCfg()
    if not mask.any():
        raise ValueError("singular system: empty mask")
    lab, seeds, _ = jump_flood_voronoi(mask)
    wts = voronoi_weights(lab, seeds, weight_scheme)
    sys_ = TonalSystem(mask, cfg, inner_cycles, inner_tol=inner_tol)
    dt = sys_.dtype
    f_arr = f.astype(dt)
    g = np.where(mask[None].astype(bool), f_arr, 0)
    seed_flat = seeds[:, 0] * mask.shape[1] + seeds[:, 1]
    m = seeds.shape[0]
    t0 = time.perf_counter()
    u, _ = inpaint(f, mask, cfg)
    u = u.astype(dt)
    cur = mse(f_arr, u)
    hist = [(0, cur, time.perf_counter() - t0, sys_.solves)]
    best_g, best, prev, steps = g.copy(), cur, cur, 0
    for k in range(1, max_steps + 1):
        for ch in range(g.shape[0]):
            delta = cell_weighted_average(lab, m, wts, f_arr[ch].astype(np.float64)
                                          - u[ch].astype(np.float64))
            gf = g[ch].ravel()
            gf[seed_flat] += (tau * delta).astype(dt)
        u = sys_.apply_B(g, warm=u)
        cur = mse(f_arr, u)
        steps = k
        hist.append((k, cur, time.perf_counter() - t0, sys_.solves))
        if cur < best:
            best, best_g = cur, g.copy()
        if stop_on_mse_increase and cur > prev:
            break
        prev = cur
    return final_state(f, mask, sys_, best_g, u, hist, steps, final_tol)


def normal_cg(sys_, rhs, cap, tol):
    """tonal.py:267-294."""
    dt = rhs.dtype
    v = np.zeros_like(rhs)
    r = rhs.copy()
    p = r.copy()
    rs = chan_dot(r, r)
    rs0 = rs.sum()
    if rs0 == 0:
        return v
    it = 0
    while it < cap and rs.sum() > tol * rs0:
        mp, _ = sys_.apply_Bt(sys_.apply_B(p))
        pmp = chan_dot(p, mp)
        alpha = np.where(pmp > 0, rs / np.where(pmp > 0, pmp, 1), 0.0)
        if not np.any(alpha > 0):
            break
        a = alpha.astype(dt)[:, None, None]
        v = v + a * p
        r = r - a * mp
        rn = chan_dot(r, r)
        beta = np.where(rs > 0, rn / np.where(rs > 0, rs, 1), 0.0)
        p = r + beta.astype(dt)[:, None, None] * p
        rs = rn
        it += 1
    return v


def ras_tonal(f, mask, init=None, cfg=None, block=64, overlap=6, local_iters=30,
              local_tol=0.1, inner_cycles=2, inner_tol=None, cold_tol=1e-4,
              local_product_tol=1e-2, rel_improvement=1e-3, max_outer=50,
              final_tol=1e-6):
    """tonal.py:309-386 (init is a final_state dict or None)."""
    cfg = cfg or SolverCfg()
    if not mask.any():
        raise ValueError("singular system: empty mask")
    sys_ = TonalSystem(mask, cfg, inner_cycles, inner_tol=inner_tol, cold_tol=cold_tol)
    dt = sys_.dtype
    f_arr = f.astype(dt)
    mb = mask[None].astype(bool)
    if init is None:
        g, u_warm = np.where(mb, f_arr, 0), None
    else:
        g, u_warm = np.where(mb, init["g"].astype(dt), 0), init["u"].astype(dt)
    w_warm = None
    h, w = mask.shape
    d = build_decomposition(h, w, block, overlap)
    nbx = d["xs"].size
    cover = np.zeros((h, w))
    for bi in range(d["nb"]):
        y0, x0 = int(d["ys"][bi // nbx]), int(d["xs"][bi % nbx])
        cover[y0:y0 + d["bh"], x0:x0 + d["bw"]] += 1.0
    inv_cover = 1.0 / cover
    blocks = []
    for bi in range(d["nb"]):
        y0, x0 = int(d["ys"][bi // nbx]), int(d["xs"][bi % nbx])
        sl = (slice(y0, y0 + d["bh"]), slice(x0, x0 + d["bw"]))
        sub = mask[sl]
        if sub.sum() == 0:
            continue
        blocks.append((sl, TonalSystem(np.ascontiguousarray(sub), cfg, inner_cycles,
                                       inner_tol=(inner_tol if inner_tol is not None
                                                  else local_product_tol))))
    t0 = time.perf_counter()
    hist = []
    best_g, best, prev, outer = g.copy(), math.inf, None, 0
    while outer < max_outer:
        u = sys_.apply_B(g, warm=u_warm)
        u_warm = u
        cur = mse(f_arr, u)
        hist.append((outer, cur, time.perf_counter() - t0, sys_.solves))
        if cur < best:
            best, best_g = cur, g.copy()
        if prev is not None and prev - cur < rel_improvement * prev:
            break
        prev = cur
        rhs, w_warm = sys_.apply_Bt(f_arr - u, warm=w_warm)
        upd = np.zeros_like(g)
        for sl, loc in blocks:
            v = normal_cg(loc, np.ascontiguousarray(rhs[:, sl[0], sl[1]]),
                          local_iters, local_tol)
            upd[:, sl[0], sl[1]] += inv_cover[sl].astype(dt) * v
        g = g + upd
        outer += 1
    total_inner = sys_.solves + sum(loc.solves for _, loc in blocks)
    st = final_state(f, mask, sys_, best_g, u_warm, hist, outer, final_tol)
    st["inner_solves"] = total_inner
    return st


def neighbor_balance_values(f, u, mask):
    """tonal.py:389-410 stored values: u + correlate(f - u, ones(3,3),
    mode="constant") / correlate(ones, ones(3,3)), cast to u's dtype, zero
    off the mask.  scipy's NI_Correlate sums the footprint in row-major
    offset order; an out-of-image tap adds cval * 1 = 0.0."""
    f = np.asarray(f, np.float64)
    u = np.asarray(u)
    diff = f - u.astype(np.float64)
    C, H, W = diff.shape
    pad = np.zeros((C, H + 2, W + 2))
    pad[:, 1:-1, 1:-1] = diff
    one = np.zeros((H + 2, W + 2))
    one[1:-1, 1:-1] = 1.0
    s = np.zeros((C, H, W))
    cnt = np.zeros((H, W))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            s = s + pad[:, 1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
            cnt = cnt + one[1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
    vals = u.astype(np.float64) + s / cnt
    return np.where(np.asarray(mask)[None] > 0, vals.astype(u.dtype), np.zeros((), u.dtype))


def cgnr_tonal(f, mask, init=None, cfg=None, rel_improvement=1e-3, max_iters=100,
               inner_cycles=1, inner_tol=None, cold_tol=1e-4, final_tol=1e-6):
    """tonal.py:198-264."""
    cfg = cfg or SolverCfg()
    if not mask.any():
        raise ValueError("singular system: empty mask")
    sys_ = TonalSystem(mask, cfg, inner_cycles, inner_tol, cold_tol=cold_tol)
    dt = sys_.dtype
    f_arr = f.astype(dt)
    mb = mask[None].astype(bool)
    if init is None:
        g, warm = np.where(mb, f_arr, 0), None
    else:
        g, warm = np.where(mb, init["g"].astype(dt), 0), init["u"].astype(dt)
    t0 = time.perf_counter()
    u = sys_.apply_B(g, warm=warm)
    r = f_arr - u
    cur = mse(f_arr, u)
    best_g, best = g.copy(), cur
    hist = [(0, cur, time.perf_counter() - t0, sys_.solves)]
    z, w_warm = sys_.apply_Bt(r)
    zs = chan_dot(z, z)
    p = z.copy()
    it, prev = 0, cur
    while it < max_iters and zs.sum() > 0:
        wv = sys_.apply_B(p)
        ws = chan_dot(wv, wv)
        alpha = np.where(ws > 0, zs / np.where(ws > 0, ws, 1), 0.0)
        a = alpha.astype(dt)[:, None, None]
        g = g + a * p
        r = r - a * wv
        cur = float(np.mean(r.astype(np.float64) ** 2))
        it += 1
        hist.append((it, cur, time.perf_counter() - t0, sys_.solves))
        if cur < best:
            best, best_g = cur, g.copy()
        if prev - cur < rel_improvement * prev:
            break
        prev = cur
        z, w_warm = sys_.apply_Bt(r, warm=w_warm)
        zn = chan_dot(z, z)
        beta = np.where(zs > 0, zn / np.where(zs > 0, zs, 1), 0.0)
        p = z + beta.astype(dt)[:, None, None] * p
        zs = zn
    return final_state(f, mask, sys_, best_g, u, hist, it, final_tol)


def run_pipeline(f, density=0.05, iterations=20, seed=0, cfg=None):
    """cli.py:206-257 with spatial='dd', tonal='ras+vi' and PipelineConfig
    defaults -> (mask, tonal state dict, spatial history, seconds)."""
    cfg = cfg or SolverCfg()
    t0 = time.perf_counter()
    mask, _, hist = delaunay_densify(f, density=density, iterations=iterations,
                                     seed=seed, cfg=cfg)
    vi = voronoi_richardson_init(f, mask, cfg)
    st = ras_tonal(f, mask, init=vi, cfg=cfg)
    return mask, st, hist, time.perf_counter() - t0


def synth(h, w, c, seed=0):
    """SURVEY.md §8d synthetic generator (integer-valued, exact in f32)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    base = (128 + 60 * np.sin(xx / 17) * np.cos(yy / 23) + 40 * (xx > 0.6 * w)
            - 30 * (yy > 0.7 * h))
    out = np.empty((c, h, w))
    for k in range(c):
        out[k] = np.clip(np.rint(base + 10 * k + rng.normal(0, 4, (h, w))), 0, 255)
    return out
