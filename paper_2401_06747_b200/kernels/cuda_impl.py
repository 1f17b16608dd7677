"""Boundary B1: the reference kernel table on sm_100a.

Same 16 names and numpy-in / numpy-out signatures as
``sparsepaint.kernels`` (kernels/__init__.py:12-29; numba_impl.py).  Each
call copies its operands to the GPU, runs the CUDA kernel through the C-ABI
and copies the result back, so the module can be monkeypatched into the
reference (test_backends.py:132-152 style) to drive the reference's own
orchestration on the GPU.  This is a parity boundary, not the performance
path (that is the device-resident B2 API of the package).
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from .._lib import call, dcode, ptr, stream

__all__ = ["negated_laplacian", "inpaint_matvec", "sym_matvec", "sym_rhs", "ct_apply",
           "sym_residual", "oras_apply", "restrict_values", "restrict_mask",
           "prolongate", "jfa_run", "jfa_dist2", "fs_dither", "assign_triangles",
           "fallback_assign", "reduce_cells"]


def _img(x):
    t = _lib.to_dev(x)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t


def _mask(m):
    return _lib.to_dev(np.asarray(m).astype(np.uint8, copy=False))


def _out(t):
    torch.cuda.current_stream().synchronize()
    return t.cpu().numpy()


def negated_laplacian(x, inv_h2):
    xt = _img(x)
    out = torch.empty_like(xt)
    c, h, w = xt.shape
    call("sp_negated_laplacian", dcode(xt), ptr(xt), ptr(out), c, h, w, float(inv_h2), stream())
    return _out(out)


def _masked(name, x, mask, inv_h2):
    xt = _img(x)
    mt = _mask(mask)
    out = torch.empty_like(xt)
    c, h, w = xt.shape
    call(name, dcode(xt), ptr(xt), ptr(mt), ptr(out), c, h, w, float(inv_h2), stream())
    return _out(out)


def inpaint_matvec(x, mask, inv_h2):
    return _masked("sp_inpaint_matvec", x, mask, inv_h2)


def sym_matvec(x, mask, inv_h2):
    return _masked("sp_sym_matvec", x, mask, inv_h2)


def sym_rhs(b, mask, inv_h2):
    return _masked("sp_sym_rhs", b, mask, inv_h2)


def ct_apply(wimg, mask, inv_h2):
    return _masked("sp_ct_apply", wimg, mask, inv_h2)


def sym_residual(u, bsym, mask, inv_h2):
    ut = _img(u)
    bt = _lib.to_dev(bsym, ut.dtype)
    mt = _mask(mask)
    r = torch.empty_like(ut)
    norms = torch.zeros(ut.shape[0], dtype=torch.float64, device=ut.device)
    c, h, w = ut.shape
    call("sp_sym_residual", dcode(ut), ptr(ut), ptr(bt), ptr(mt), ptr(r), ptr(norms), c, h, w,
         float(inv_h2), stream())
    return _out(r), _out(norms)


def oras_apply(u, r, mask, xs, ys, bh, bw, gamma, taus, cap, weights, inv_h2):
    """Mutates the numpy array ``u`` in place (numba_impl.py:161-263)."""
    ut = _img(u)
    rt = _lib.to_dev(r, ut.dtype)
    mt = _mask(mask)
    wt = _lib.to_dev(weights, ut.dtype)
    xs_h = np.ascontiguousarray(xs, np.int64)
    ys_h = np.ascontiguousarray(ys, np.int64)
    taus_h = np.ascontiguousarray(taus, np.float64)
    c, h, w = ut.shape
    call("sp_oras_apply", dcode(ut), ptr(ut), ptr(rt), ptr(mt), ptr(xs_h), xs_h.size,
         ptr(ys_h), ys_h.size, int(bh), int(bw), float(gamma), ptr(taus_h), int(cap),
         ptr(wt), float(inv_h2), c, h, w, stream())
    u[...] = _out(ut)


def restrict_values(fine):
    ft = _img(fine)
    c, h, w = ft.shape
    out = torch.empty((c, (h + 1) // 2, (w + 1) // 2), dtype=ft.dtype, device=ft.device)
    call("sp_restrict_values", dcode(ft), ptr(ft), ptr(out), c, h, w, stream())
    return _out(out)


def restrict_mask(mask, values):
    mt = _mask(mask)
    vt = _img(values)
    c = vt.shape[0]
    h, w = mt.shape
    cm = torch.empty(((h + 1) // 2, (w + 1) // 2), dtype=torch.uint8, device=mt.device)
    cv = torch.empty((c,) + tuple(cm.shape), dtype=vt.dtype, device=vt.device)
    call("sp_restrict_mask", dcode(vt), ptr(mt), ptr(vt), ptr(cm), ptr(cv), c, h, w, stream())
    return _out(cm), _out(cv)


def prolongate(coarse, h, w):
    ct = _img(coarse)
    c, ch, cw = ct.shape
    out = torch.empty((c, h, w), dtype=ct.dtype, device=ct.device)
    call("sp_prolongate", dcode(ct), ptr(ct), ptr(out), c, ch, cw, int(h), int(w), stream())
    return _out(out)


def jfa_run(labels, seeds, steps):
    lt = _lib.to_dev(np.asarray(labels).astype(np.int32, copy=False))
    st = _lib.to_dev(np.asarray(seeds).astype(np.int64, copy=False).reshape(-1, 2))
    steps_h = np.ascontiguousarray(steps, np.int64)
    out = torch.empty_like(lt)
    h, w = lt.shape
    call("sp_jfa_run", ptr(lt), ptr(out), ptr(st), st.shape[0], ptr(steps_h), steps_h.size, h, w,
         stream())
    return _out(out)


def jfa_dist2(labels, seeds):
    lt = _lib.to_dev(np.asarray(labels).astype(np.int32, copy=False))
    st = _lib.to_dev(np.asarray(seeds).astype(np.int64, copy=False).reshape(-1, 2))
    out = torch.empty(lt.shape, dtype=torch.int64, device=lt.device)
    h, w = lt.shape
    call("sp_jfa_dist2", ptr(lt), ptr(st), st.shape[0], ptr(out), h, w, None, stream())
    return _out(out)


def fs_dither(dens):
    dt = _lib.to_dev(np.asarray(dens, np.float64))
    out = torch.empty(dt.shape, dtype=torch.uint8, device=dt.device)
    h, w = dt.shape
    call("sp_fs_dither", ptr(dt), ptr(out), h, w, stream())
    return _out(out)


def assign_triangles(tris, vy, vx, h, w):
    tt = _lib.to_dev(np.asarray(tris).astype(np.int64, copy=False).reshape(-1, 3))
    vyt = _lib.to_dev(np.asarray(vy).astype(np.int64, copy=False))
    vxt = _lib.to_dev(np.asarray(vx).astype(np.int64, copy=False))
    out = torch.empty((int(h), int(w)), dtype=torch.int32, device=tt.device)
    call("sp_assign_triangles", ptr(tt), tt.shape[0], ptr(vyt), ptr(vxt), int(h), int(w),
         ptr(out), stream())
    return _out(out)


def fallback_assign(assign, labels, seed_min_tri):
    at = _lib.to_dev(np.asarray(assign).astype(np.int32, copy=False))
    lt = _lib.to_dev(np.asarray(labels).astype(np.int32, copy=False))
    st = _lib.to_dev(np.asarray(seed_min_tri).astype(np.int32, copy=False))
    out = torch.empty_like(at)
    h, w = at.shape
    call("sp_fallback_assign", ptr(at), ptr(lt), ptr(st), ptr(out), h, w, stream())
    return _out(out)


def reduce_cells(assign, err, ntris):
    at = _lib.to_dev(np.asarray(assign).astype(np.int32, copy=False))
    et = _lib.to_dev(np.asarray(err, np.float64))
    n = int(ntris)
    sums = torch.zeros(n, dtype=torch.float64, device=at.device)
    ai = torch.full((n,), -1, dtype=torch.int64, device=at.device)
    av = torch.full((n,), -1.0, dtype=torch.float64, device=at.device)
    h, w = at.shape
    if n:
        call("sp_reduce_cells", ptr(at), ptr(et), n, ptr(sums), ptr(ai), ptr(av), h, w, stream())
    return _out(sums), _out(ai), _out(av)
