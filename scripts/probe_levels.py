"""Per-level cost of a warm 4K RGB V-cycle: time 20 warm V-cycles with the
hierarchy truncated to L levels (L = 1 .. full).  The difference between
consecutive L approximates what level L (and its launches) adds.  Also the
pipeline with the device-driven tolerance loop on / off.

    python scripts/probe_levels.py [--pipeline]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_06747_b200 as sp
from oracle import oracle as O
from paper_2401_06747_b200 import _lib

H, W, C = 2160, 3840, 3
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
full = None
prev = 0.0
for L in range(1, 10):
    cfg = sp.MultigridConfig(tol=None, cycles=20, levels=L)
    sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
    t = time.perf_counter()
    sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 20 * 1e3
    print(f"levels {L}: {ms:.3f} ms per V-cycle (+{ms - prev:.3f})", flush=True)
    prev = ms
if "--pipeline" in sys.argv:
    pc = sp.PipelineConfig()
    fd = torch.from_numpy(f).cuda()
    for loop in (0, 1, 0, 1):
        _lib.load().sp_graph_loop(loop)
        for _ in range(2):
            sp.run_pipeline(sp.Image(fd), pc)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            m, st, hist, _ = sp.run_pipeline(sp.Image(fd), pc)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"graph_loop={loop}: pipeline {e0.elapsed_time(e1) / 3:.1f} ms mse {st.mse:.6f}",
              flush=True)
