"""ORAS local CG statistics for one cold 4K inpaint + 2 warm V-cycles."""
import sys, os, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200._lib import call
from oracle import oracle as O
H, W, C = 2160, 3840, 3
f = O.synth(H, W, C, 0)
for dens in (0.05, 0.0024):
    mask = (np.random.default_rng(2).random((H, W)) < dens).astype(np.uint8)
    fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
    u, rep = sp.inpaint(fi, mi)
    st = (ctypes.c_uint64 * 4)()
    call("sp_stats", 1, None)
    u2, rep = sp.inpaint(fi, mi, sp.MultigridConfig(tol=None, cycles=2), init=u)
    torch.cuda.synchronize()
    call("sp_stats", 0, st)
    print(f"density {dens}: jobs={st[0]} iters={st[1]} mean={st[1]/max(1,st[0]):.2f} "
          f"zero-iter={st[2]/max(1,st[0]):.2%} max={st[3]}")
