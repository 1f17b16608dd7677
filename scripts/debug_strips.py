import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200.strips import StripSolver
from oracle import oracle as O
c, h, w = 3, 1024, 1536
f = O.synth(h, w, c, 0)
mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
for cyc in (1, 2, 3):
    res = {}
    for P in (1, 2, 4):
        s = StripSolver(h, w, c, strips=P, cfg=sp.MultigridConfig(tol=None, cycles=cyc), La=3)
        u, rep = s.inpaint(sp.Image(f), sp.Mask(mask))
        res[P] = u.data
    for P in (2, 4):
        d = np.abs(res[P] - res[1])
        rows = np.nonzero(d.max(axis=(0, 2)))[0]
        print(f"cycles {cyc} P {P}: maxdiff {d.max():.3e} rows {rows[:10]} .. {rows[-5:] if rows.size else ''} n={rows.size}", flush=True)
for P in (1, 2):
    s = StripSolver(h, w, c, strips=P, cfg=sp.MultigridConfig(tol=1e-6, max_cycles=60), La=3)
    u, rep = s.inpaint(sp.Image(f), sp.Mask(mask))
    print(P, rep.iterations, rep.residuals[:4], rep.residuals[-2:])
