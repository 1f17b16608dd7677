"""Quick perf probe: finest-level kernel timings (sp_hier_bench), warm 4K RGB
V-cycle time, and the pipeline step time (device events).

    python scripts/probe_perf.py [--no-pipeline] [sp_switch=value ...]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_06747_b200 as sp
from oracle import oracle as O
from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200.solver import GridHierarchy, MultigridConfig, _masked_rhs

import subprocess
import threading

H, W, C = 2160, 3840, 3
_clk = []


def _sample():
    while not _done:
        try:
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            _clk.append(out)
        except Exception:
            pass
        time.sleep(0.5)


for a in sys.argv[1:]:
    if "=" in a:
        k, v = a.split("=")
        getattr(_lib.load(), k)(int(v))
_done = False
threading.Thread(target=_sample, daemon=True).start()
PEAK = 6544.0
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fd = torch.from_numpy(f).cuda()
fi, mi = sp.Image(fd), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
names = ["resid", "oras", "blend", "resid<1>", "prolong"]
hier = GridHierarchy.build(mi, sp.Image(fd.float()), MultigridConfig(), channels=C)
bsym = _masked_rhs(fd.float().contiguous(), mi.tensor())
hier.solve_sym(bsym, tol=1e-4, cascade=True)
for which in range(5):
    t_ms, nbytes = ctypes.c_double(), ctypes.c_double()
    _lib.call("sp_hier_bench", hier._h, which, 20, ctypes.byref(t_ms), ctypes.byref(nbytes),
              _lib.stream())
    gbs = nbytes.value / (t_ms.value * 1e-3) / 1e9
    print(f"{names[which]:10s} {t_ms.value * 1e3:8.1f} us {nbytes.value / 1e6:8.1f} MB "
          f"{gbs:7.0f} GB/s frac {gbs / PEAK:.3f}", flush=True)
del hier
cfg = sp.MultigridConfig(tol=None, cycles=10)
sp.inpaint(fi, mi, cfg, init=u)
torch.cuda.synchronize()
t = time.perf_counter()
sp.inpaint(fi, mi, cfg, init=u)
torch.cuda.synchronize()
print(f"V-cycle {(time.perf_counter() - t) * 1e2:.3f} ms (10 warm cycles)", flush=True)
if "--no-pipeline" not in sys.argv:
    pc = sp.PipelineConfig()
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
    print(f"pipeline {e0.elapsed_time(e1) / 3:.1f} ms  mse {st.mse:.6f} dd {hist[-1][2]:.6f} "
          f"count {m.count}", flush=True)
_done = True
print("clocks (sm, max, W):", _clk[len(_clk) // 2] if _clk else None, "samples", len(_clk))
