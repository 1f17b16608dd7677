"""End-to-end probe: GPU pipeline vs CPU oracle at a small size, then timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from oracle import oracle as O

def run(h, w, c, oracle=True, reps=1):
    f = O.synth(h, w, c, 0)
    cfg = sp.PipelineConfig()
    for r in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        mask, st, hist, sec = sp.run_pipeline(sp.Image(f), cfg)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"GPU {h}x{w}x{c}: {dt:.3f}s  mask={mask.count} dd_mse={hist[-1][2]:.6f} final_mse={st.mse:.6f} "
              f"ras_outer={st.iterations}", flush=True)
    if oracle:
        t = time.perf_counter()
        m2, st2, h2, _ = O.run_pipeline(f)
        print(f"CPU {h}x{w}x{c}: {time.perf_counter()-t:.2f}s mask={int(m2.sum())} dd_mse={h2[-1][2]:.6f} "
              f"final_mse={st2['mse']:.6f} ras_outer={st2['iterations']}  mask_diff={int((m2 != mask.indicator).sum())}",
              flush=True)

for args in sys.argv[1:] or ["64,64,3,1", "128,128,1,1"]:
    h, w, c, o = (int(x) for x in args.split(","))
    run(h, w, c, bool(o), reps=2 if not o else 1)
