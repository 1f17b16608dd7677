"""Where the end-to-end (host image in, host mask/values out) time goes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from oracle.oracle import synth
f_host = synth(2160, 3840, 3, 0)
f_pin = torch.from_numpy(f_host).pin_memory()
f_dev = f_pin.cuda()
cfg = sp.PipelineConfig()
for _ in range(2):
    sp.run_pipeline(sp.Image(f_dev), cfg)
torch.cuda.synchronize()
for rep in range(3):
    T = {}
    t = time.perf_counter()
    img = sp.Image(f_pin); d = img.tensor(); torch.cuda.synchronize(); T["h2d"] = time.perf_counter() - t
    t = time.perf_counter()
    m, st, h, _ = sp.run_pipeline(sp.Image(d), cfg); torch.cuda.synchronize(); T["pipeline"] = time.perf_counter() - t
    t = time.perf_counter(); mi = m.indicator; T["mask_d2h"] = time.perf_counter() - t
    t = time.perf_counter(); g = st.g.data; T["g_d2h"] = time.perf_counter() - t
    t = time.perf_counter()
    m2, st2, h2, _ = sp.run_pipeline(sp.Image(f_pin), cfg); mi2 = m2.indicator; g2 = st2.g.data
    T["e2e_total"] = time.perf_counter() - t
    print({k: round(v * 1e3, 1) for k, v in T.items()}, g.dtype, g.shape, flush=True)
