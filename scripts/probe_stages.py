"""Stage breakdown of the 4K pipeline (host timers around device-synced calls)."""
import sys, os, time, collections, functools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import spatial, tonal, solver, geometry
from oracle import oracle as O

T = collections.defaultdict(float); N = collections.Counter()
def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    @functools.wraps(fn)
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); T[label or name] += time.perf_counter() - t; N[label or name] += 1
        return r
    setattr(mod, name, w)

wrap(solver.InpaintSolver, "inpaint", "inpaint(all)")
wrap(geometry.GeoWorkspace, "voronoi"); wrap(geometry.GeoWorkspace, "delaunay")
wrap(geometry.GeoWorkspace, "accumulate"); wrap(geometry.GeoWorkspace, "select")
wrap(spatial, "_analytic_mask_t", "init_mask")
wrap(tonal._RasBlocks, "normal_cg", "ras_local_cg"); wrap(tonal._RasBlocks, "__init__", "ras_blocks_init")
wrap(tonal._TonalSystem, "apply_B"); wrap(tonal._TonalSystem, "apply_Bt")
wrap(tonal, "_final_state")
wrap(sp.pipeline, "run_spatial"); wrap(sp.pipeline, "run_tonal")
wrap(tonal, "voronoi_richardson_init", "vi(total)"); wrap(tonal, "ras_tonal", "ras(total)")
h, w, c = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2160,3840,3").split(","))
f = O.synth(h, w, c, 0)
cfg = sp.PipelineConfig()
sp.run_pipeline(sp.Image(f), cfg)
T.clear(); N.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
mask, st, hist, sec = sp.run_pipeline(sp.Image(f), cfg)
torch.cuda.synchronize(); tot = time.perf_counter() - t0
print(f"total {tot:.3f}s")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"  {k:22s} {v*1e3:9.1f} ms  n={N[k]}")
