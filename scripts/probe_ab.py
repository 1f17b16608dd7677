"""A/B of the ORAS local-CG variants on a warm 4K RGB V-cycle + stats."""
import sys, os, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200._lib import call
from oracle import oracle as O
H, W, C = 2160, 3840, 3
f = O.synth(H, W, C, 0)
lib = _lib.load()
for dens in (0.05, 0.0024):
    mask = (np.random.default_rng(2).random((H, W)) < dens).astype(np.uint8)
    fi, mi = sp.Image(torch.from_numpy(f).cuda()), sp.Mask(torch.from_numpy(mask).cuda())
    u, rep = sp.inpaint(fi, mi)
    VARS = [tuple(map(int, a.split(':'))) for a in sys.argv[1:]] or [(0, 2), (4, 2), (0, 2), (4, 2)]
    for var, mv in VARS:
        lib.sp_oras_variant(var)
        lib.sp_march_variant(mv)
        sp.solver._POOL.clear()
        cfg = sp.MultigridConfig(tol=None, cycles=10)
        u2, rep = sp.inpaint(fi, mi, cfg, init=u)
        torch.cuda.synchronize(); t = time.perf_counter()
        u2, rep = sp.inpaint(fi, mi, cfg, init=u)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        st = (ctypes.c_uint64 * 4)()
        call("sp_stats", 1, None)
        sp.inpaint(fi, mi, sp.MultigridConfig(tol=None, cycles=1), init=u)
        torch.cuda.synchronize()
        call("sp_stats", 0, st)
        print(f"dens {dens} oras {var} march {mv}: {dt*1e2:.3f} ms/V-cycle; jobs={st[0]} "
              f"mean iters={st[1]/max(1,st[0]):.2f} zero={st[2]/max(1,st[0]):.2%} max={st[3]}",
              flush=True)
    lib.sp_oras_variant(0)
    lib.sp_march_variant(2)
