"""RAS local normal-CG batch statistics on the 4K pipeline: active tiles and
V-cycles per CG iteration (per-tile stopping tail)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import tonal
from oracle import oracle as O

log = []
orig_solve = tonal._RasBlocks._solve
def _solve(self, bsym, active_h):
    torch.cuda.synchronize(); t = time.perf_counter()
    u = orig_solve(self, bsym, active_h)
    torch.cuda.synchronize()
    log.append((int(active_h.sum()), int(self._iters[active_h > 0].max()) if active_h.any() else 0,
                float(np.mean(self._iters[active_h > 0])) if active_h.any() else 0, time.perf_counter() - t))
    return u
tonal._RasBlocks._solve = _solve
f = O.synth(2160, 3840, 3, 0)
cfg = sp.PipelineConfig()
sp.run_pipeline(sp.Image(f), cfg)
log.clear()
sp.run_pipeline(sp.Image(f), cfg)
print("solves:", len(log), "total ms", sum(x[3] for x in log) * 1e3)
for i, (na, mx, mean, dt) in enumerate(log):
    print(f"{i:3d} active {na:5d} vcycles max {mx:3d} mean {mean:5.2f}  {dt*1e3:7.2f} ms")
