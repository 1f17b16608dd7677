"""Kernel breakdown of the RAS local normal-CG (tonal.py:267-294 batched) on the 4K pipeline."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import tonal
from oracle.oracle import synth
f = torch.from_numpy(synth(2160, 3840, 3, 0)).cuda()
cfg = sp.PipelineConfig()
sp.run_pipeline(sp.Image(f), cfg)
prof_on = [None]
orig = tonal._RasBlocks.normal_cg
evs = []
def ncg(self, *a, **k):
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        v = orig(self, *a, **k)
        torch.cuda.synchronize()
    evs.append(p)
    return v
tonal._RasBlocks.normal_cg = ncg
sp.run_pipeline(sp.Image(f), cfg)
tot = collections.defaultdict(float); n = collections.Counter(); span = 0.0
for p in evs:
    lo, hi = float("inf"), 0.0
    for e in p.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        tot[name] += e.device_time_total; n[name] += 1
        lo = min(lo, e.time_range.start); hi = max(hi, e.time_range.end)
    span += hi - lo
T = sum(tot.values())
print(f"# RAS normal_cg x{len(evs)}: kernel time {T/1e3:.1f} ms, span {span/1e3:.1f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{k[:72]:72s} {v/1e3:9.2f} {v/T:7.1%} {n[k]:6d} {v/n[k]:8.1f}")
