"""Deterministic device reductions and elementwise helpers (vec.cu)."""

from __future__ import annotations

import torch

from ._lib import call, dcode, ptr, stream


def chan_reduce(mode, x, y=None, z=None, channels=None):
    """Per-channel double sums over the planes of x (see sp_chan_reduce)."""
    C = x.shape[0] if channels is None else channels
    n = x.numel() // C
    out = torch.empty(C, dtype=torch.float64, device=x.device)
    if y is not None and y.dtype != x.dtype:
        y = y.to(x.dtype)
    if z is not None and z.dtype != torch.float64:
        z = z.to(torch.float64)
    # bind the contiguous copies so they outlive the (asynchronous) launch
    xc = x.contiguous()
    yc = None if y is None else y.contiguous()
    zc = None if z is None else z.contiguous()
    call("sp_chan_reduce", dcode(xc), mode, ptr(xc), ptr(yc), ptr(zc), n, C, ptr(out),
         stream())
    return out


def chan_dot(a, b):
    """tonal.py:91-97: per-channel double dot products (device tensor)."""
    return chan_reduce(1, a, b)


def sumsq(a, channels=1):
    return chan_reduce(0, a, channels=channels)


def sq_err(x, z):
    """sum over everything of (x - z)^2 in double (device scalar tensor)."""
    return chan_reduce(2, x, z=z, channels=1)


def mse_t(a, b) -> float:
    """MSE over all channels in double (grid.py:188-193, tonal.py:86-88)."""
    if a.dtype == b.dtype and a.dtype in (torch.float32, torch.float64):
        # both widened exactly in the kernel: no f64 copy of either
        return float(chan_reduce(3, a, y=b, channels=1).item()) / max(1, a.numel())
    if a.dtype == torch.float64 and b.dtype != torch.float64:
        a, b = b, a
    x = a if a.dtype in (torch.float32, torch.float64) else a.to(torch.float64)
    return float(sq_err(x, b).item()) / max(1, x.numel())


def error_map(u, f64, with_sum=False):
    """spatial.py:184-186: sum_c (u - f)^2 in double -> (H, W).  with_sum:
    also the total of the map (a device double, the MSE numerator) from the
    same pass."""
    C, H, W = u.shape
    e = torch.empty((H, W), dtype=torch.float64, device=u.device)
    if not with_sum:
        call("sp_error_map", dcode(u), ptr(u), ptr(f64), ptr(e), C, H * W, stream())
        return e
    tot = torch.empty((), dtype=torch.float64, device=u.device)
    call("sp_error_map_sum", dcode(u), ptr(u), ptr(f64), ptr(e), C, H * W, ptr(tot), stream())
    return e, tot
