"""Per-kernel device-time breakdown of one warm 4K RGB pipeline step via the
CUDA activity trace (torch.profiler / CUPTI: every kernel of the process,
including libsparsepaint_b200.so's, with concurrent-kernel timestamps).

    python scripts/kprof.py [H,W,C] > gpurun_out/kprof.txt
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2401_06747_b200 as sp
from oracle.oracle import synth

h, w, c = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2160,3840,3").split(","))
f = torch.from_numpy(synth(h, w, c, 0)).cuda()
cfg = sp.PipelineConfig()
for _ in range(2):
    sp.run_pipeline(sp.Image(f), cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
sp.run_pipeline(sp.Image(f), cfg)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sp.run_pipeline(sp.Image(f), cfg)
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
n = collections.Counter()
span = [float("inf"), 0.0]
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    d = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    tot[name] += d
    n[name] += 1
    span[0] = min(span[0], e.time_range.start)
    span[1] = max(span[1], e.time_range.end)
T = sum(tot.values())
print(f"# {h}x{w}x{c} pipeline: wall {wall * 1e3:.1f} ms (unprofiled); "
      f"kernel time {T / 1e3:.1f} ms over {sum(n.values())} device ops; "
      f"trace span {(span[1] - span[0]) / 1e3:.1f} ms")
print(f"{'kernel':72s} {'ms':>9s} {'share':>7s} {'n':>6s} {'avg_us':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:45]:
    print(f"{k[:72]:72s} {v / 1e3:9.2f} {v / T:7.1%} {n[k]:6d} {v / n[k]:8.1f}")
