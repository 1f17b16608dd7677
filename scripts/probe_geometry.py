"""Densification geometry at 4K: per-stage device time (CUDA events) of the
JFA Voronoi, Delaunay corner scan + unique, the triangle-bucket accumulate
(tiled default vs the global-atomic + sort path) and the pick selection, on
a 0.24% (densification iteration 0) and a 5% (last iteration) random mask.

    python scripts/probe_geometry.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200.geometry import workspace

H, W = 2160, 3840
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lib = _lib.load()
rng = np.random.default_rng(0)
err = torch.from_numpy(rng.random((H, W)) * 50.0).cuda()
s = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for dens in (0.0024, 0.05):
    m = torch.from_numpy((rng.random((H, W)) < dens).astype(np.uint8)).cuda()
    ws = workspace(H, W)
    t_vor = timed(lambda: ws.voronoi(m, None))
    ws.voronoi(m, None)
    t_vor_h = timed(lambda: ws.voronoi(m, ws.max_radius))
    t_del = timed(lambda: ws.delaunay())
    nb = ws.delaunay()
    out = {}
    for mode in (0, 1):
        lib.sp_geo_accumulate_mode(mode)
        out[mode] = timed(lambda: ws.accumulate(err))
        sums, amax, _ = ws.buckets(nb)
        out[f"chk{mode}"] = (float(sums.sum()), int(amax.sum()))
    lib.sp_geo_accumulate_mode(1)
    mk = m.clone()
    t_sel = timed(lambda: ws.select(mk.copy_(m), nb, 20000))
    print(f"density {dens}: seeds {ws.m} tris {nb} | voronoi {t_vor:.3f} ms (hinted "
          f"{t_vor_h:.3f}) | delaunay {t_del:.3f} ms | accumulate tiled {out[1]:.3f} ms vs "
          f"atomic+sort {out[0]:.3f} ms (same: {out['chk0'] == out['chk1']}) | select "
          f"{t_sel:.3f} ms", flush=True)

# per-kernel breakdown of one tiled accumulate per density (CUPTI)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
for dens in (0.0024, 0.05):
    m = torch.from_numpy((rng.random((H, W)) < dens).astype(np.uint8)).cuda()
    ws = workspace(H, W)
    ws.voronoi(m, None)
    nb = ws.delaunay()
    ws.accumulate(err)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ws.accumulate(err)
        torch.cuda.synchronize()
    rows = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            rows.append((e.name.split("(")[0][:60], e.device_time_total))
    print(f"density {dens} accumulate kernels:", ", ".join(f"{n} {t:.1f}us" for n, t in rows),
          flush=True)
