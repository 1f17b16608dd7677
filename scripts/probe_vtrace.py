"""Kernel-by-kernel trace of ONE warm 4K RGB V-cycle (CUPTI via
torch.profiler): name, duration and the gap before each kernel, in order.

    python scripts/probe_vtrace.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2401_06747_b200 as sp
from oracle import oracle as O

H, W, C = 2160, 3840, 3
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
cfg = sp.MultigridConfig(tol=None, cycles=1)
for _ in range(3):
    sp.inpaint(fi, mi, cfg, init=u)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
prev = None
tot = 0.0
for e in ev:
    name = e.name.replace("(anonymous namespace)::", "").split("(")[0][:60]
    gap = 0.0 if prev is None else e.time_range.start - prev
    dur = e.time_range.end - e.time_range.start
    tot += dur
    print(f"{name:60s} {dur:8.1f} us  gap {gap:6.1f}")
    prev = e.time_range.end
print(f"sum of kernel durations {tot:.1f} us, span {ev[-1].time_range.end - ev[0].time_range.start:.1f} us")
