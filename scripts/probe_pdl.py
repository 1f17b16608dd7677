"""Warm 4K RGB V-cycle time and pipeline time vs the first multigrid level
launched with programmatic dependent launch (sp_pdl_from_level).

    python scripts/probe_pdl.py [--pipeline]
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
from paper_2401_06747_b200.solver import _POOL

H, W, C = 2160, 3840, 3
lib = _lib.load()
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fd = torch.from_numpy(f).cuda()
fi, mi = sp.Image(fd), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
ref = None
for frm in (-1, 5, 4, 3, 2, 1, 0, -1):
    lib.sp_pdl_from_level(frm)
    _POOL.clear()
    cfg = sp.MultigridConfig(tol=None, cycles=20)
    out, _ = sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out, _ = sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 20 * 1e3
    same = ref is None or torch.equal(out.tensor(), ref)
    ref = out.tensor().clone() if ref is None else ref
    print(f"pdl from level {frm:2d}: {ms:.3f} ms per V-cycle, identical {same}", flush=True)
if "--pipeline" in sys.argv:
    pc = sp.PipelineConfig()
    for frm in (-1, 3, -1, 3, 1):
        lib.sp_pdl_from_level(frm)
        _POOL.clear()
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
        print(f"pdl from {frm:2d}: pipeline {e0.elapsed_time(e1) / 3:.1f} ms mse {st.mse:.6f}",
              flush=True)
