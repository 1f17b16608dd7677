"""4K RGB pipeline device time (CUDA events) per ORAS kernel variant, the
other switches left at their defaults: python scripts/probe_oras_pipe.py 7 8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2401_06747_b200 as sp
from oracle.oracle import synth
from paper_2401_06747_b200 import _lib

lib = _lib.load()
f = torch.from_numpy(synth(2160, 3840, 3, 0)).cuda()
cfg = sp.PipelineConfig()
variants = [int(a) for a in sys.argv[1:]] or [7, 8]
for v in variants * 2:
    lib.sp_oras_variant(v)
    sp.solver._POOL.clear()
    sp.run_pipeline(sp.Image(f), cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg)
    e1.record()
    torch.cuda.synchronize()
    print(f"oras {v}: {e0.elapsed_time(e1) / 3:.2f} ms/pipeline  mse={st.mse:.9f} "
          f"count={mask.count} hist={len(hist)}", flush=True)
