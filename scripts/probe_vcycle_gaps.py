"""Kernel time vs span of warm 4K V-cycles (CUPTI trace): how much of a
V-cycle is inter-kernel gap, and how the time splits by level size."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2401_06747_b200 as sp
from oracle import oracle as O
H, W, C, N = 2160, 3840, 3, 10
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
cfg = sp.MultigridConfig(tol=None, cycles=N)
sp.inpaint(fi, mi, cfg, init=u)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
ev = sorted([e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
ks = [e for e in ev if "sp::" in e.name]
span = ks[-1].time_range.end - ks[0].time_range.start
busy = sum(e.device_time_total for e in ks)
short = [e for e in ks if e.device_time_total < 8.0]
print(f"{N} V-cycles: span {span/1e3:.2f} ms, kernel busy {busy/1e3:.2f} ms, "
      f"{len(ks)} kernels ({len(ks)/N:.0f}/cycle), short(<8us) {len(short)} = {sum(e.device_time_total for e in short)/1e3:.2f} ms")
gaps = [ks[i+1].time_range.start - ks[i].time_range.end for i in range(len(ks)-1)]
gaps = [g for g in gaps if g > 0]
print(f"gaps: total {sum(gaps)/1e3:.2f} ms, median {sorted(gaps)[len(gaps)//2]:.2f} us")
