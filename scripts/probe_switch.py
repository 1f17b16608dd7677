"""4K RGB pipeline device time (CUDA events) per setting of the library's
A/B switches, the rest at their defaults; each setting runs twice, interleaved:

    python scripts/probe_switch.py sp_spec_vcycle=0 sp_spec_vcycle=1
    python scripts/probe_switch.py sp_oras_variant=7 sp_oras_variant=8,sp_tile_list=0
"""
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
settings = [[kv.split("=") for kv in a.split(",")] for a in sys.argv[1:]]
defaults = {k: getattr(lib, k)(-1) for s in settings for k, _ in s}
for st in settings * 2:
    for k, v in defaults.items():
        getattr(lib, k)(v)
    for k, v in st:
        getattr(lib, k)(int(v))
    sp.solver._POOL.clear()
    sp.run_pipeline(sp.Image(f), cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        mask, stt, hist, _ = sp.run_pipeline(sp.Image(f), cfg)
    e1.record()
    torch.cuda.synchronize()
    name = ",".join(f"{k}={v}" for k, v in st)
    print(f"{name}: {e0.elapsed_time(e1) / 3:.2f} ms/pipeline  mse={stt.mse:.9f} "
          f"count={mask.count}", flush=True)
