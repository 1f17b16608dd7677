"""Quick GPU probe: 4K RGB inpaint timing + per-V-cycle time."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from oracle import oracle as O

H, W, C = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (2160, 3840, 3)))
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    u, rep = sp.inpaint(fi, mi)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"cold inpaint {H}x{W}x{C}: {dt*1e3:.2f} ms, cycles={rep.iterations}, res={rep.residuals[-1]:.3e}")
cfg = sp.MultigridConfig(tol=None, cycles=10)
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    u2, rep = sp.inpaint(fi, mi, cfg, init=u)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"10 warm V-cycles: {dt*1e3:.2f} ms -> {dt*1e2:.3f} ms/V-cycle")
