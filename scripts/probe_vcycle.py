"""One warm-up solve, then N warm V-cycles (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from oracle import oracle as O
H, W, C, N = 2160, 3840, 3, int(sys.argv[1]) if len(sys.argv) > 1 else 1
f = O.synth(H, W, C, 0)
mask = (np.random.default_rng(2).random((H, W)) < 0.05).astype(np.uint8)
fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
u, rep = sp.inpaint(fi, mi)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("warm")
u2, rep = sp.inpaint(fi, mi, sp.MultigridConfig(tol=None, cycles=N), init=u)
torch.cuda.synchronize()
