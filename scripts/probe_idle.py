"""GPU idle gaps of one warm 4K pipeline step (CUPTI trace): total idle and
the kernels that precede the largest gaps (= where the host synchronises)."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2401_06747_b200 as sp
from oracle.oracle import synth
f = torch.from_numpy(synth(2160, 3840, 3, 0)).cuda()
cfg = sp.PipelineConfig()
for _ in range(2):
    sp.run_pipeline(sp.Image(f), cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    sp.run_pipeline(sp.Image(f), cfg)
    torch.cuda.synchronize()
ev = sorted([e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
name = lambda e: e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
idle = collections.defaultdict(float); cnt = collections.Counter()
end = ev[0].time_range.end
tot = 0.0
for a, b in zip(ev, ev[1:]):
    end = max(end, a.time_range.end)
    g = b.time_range.start - end
    if g > 5:
        key = f"{name(a)} -> {name(b)}"
        idle[key] += g; cnt[key] += 1; tot += g
print(f"span {(ev[-1].time_range.end - ev[0].time_range.start)/1e3:.1f} ms, idle (gaps > 5 us) {tot/1e3:.1f} ms")
for k, v in sorted(idle.items(), key=lambda z: -z[1])[:25]:
    print(f"{v/1e3:7.2f} ms {cnt[k]:5d}  {k}")
