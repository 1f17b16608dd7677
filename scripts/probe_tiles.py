"""Batched RAS block-local products (tonal.py:120-131) on a 4K-like block
set: time per apply_B for the fused tile solver vs the batched hierarchy."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import tonal, _lib
from oracle import oracle as O
lib = _lib.load()
H, W, C = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1080,1920,3").split(","))
modes = [int(x) for x in sys.argv[2:]] or [1, 0]
mask = (np.random.default_rng(9).random((H, W)) < 0.05).astype(np.uint8)
for tf in modes:
    lib.sp_tile_fused(tf)
    sp.solver._POOL.clear()
    blocks = tonal._RasBlocks(torch.from_numpy(mask).cuda(), sp.InpaintSolver(), C, sp.RasTonalConfig())
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((blocks.nt, C, blocks.bh, blocks.bw))).float().cuda()
    act = np.ones(blocks.nt, np.int32); act_d = torch.from_numpy(act).cuda()
    blocks.apply_B(x, act, act_d); torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("warm")
    t = time.perf_counter()
    for _ in range(3):
        blocks.apply_B(x, act, act_d)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"tile_fused {tf}: {blocks.nt} blocks x {C} ch: {(time.perf_counter()-t)/3*1e3:.2f} ms per apply_B, "
          f"V-cycles {blocks._iters.mean():.2f}", flush=True)
if os.environ.get("KPROF"):
    import collections
    from torch.profiler import ProfilerActivity, profile
    lib.sp_tile_fused(1)
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        blocks.apply_B(x, act, act_d); torch.cuda.synchronize()
    tot = collections.defaultdict(float); n = collections.Counter()
    for e in p.events():
        if e.device_type != torch.autograd.DeviceType.CUDA: continue
        k = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        tot[k] += e.device_time_total; n[k] += 1
    for k, v in sorted(tot.items(), key=lambda z: -z[1])[:12]:
        print(f"{k[:60]:60s} {v/1e3:8.3f} ms {n[k]:4d} {v/n[k]:8.1f} us")
