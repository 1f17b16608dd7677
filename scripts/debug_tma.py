import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200.solver import GridHierarchy, _masked_rhs, _POOL
from oracle import oracle as O
lib = _lib.load()
for (c, h, w) in [(1, 128, 128), (1, 200, 256), (3, 130, 384)]:
    f = O.synth(h, w, c, 0)
    mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
    ft = torch.from_numpy(f).float().cuda(); mt = torch.from_numpy(mask).cuda()
    u0 = ft + torch.randn_like(ft)
    bsym = _masked_rhs(ft, mt)
    res = {}
    for v in (0, 2):
        lib.sp_march_variant(v); _POOL.clear()
        hier = GridHierarchy.build(sp.Mask(mt), sp.Image(ft), sp.MultigridConfig())
        hier.solve_sym(bsym, init=u0, tol=1e9)
        r = torch.empty_like(ft); nrm = torch.empty(c, dtype=torch.float64, device="cuda")
        _lib.call("sp_hier_residual", hier._h, 0, _lib.ptr(r), _lib.ptr(nrm), _lib.stream())
        torch.cuda.synchronize()
        res[v] = (r.cpu().numpy(), nrm.cpu().numpy())
    d = res[0][0] != res[2][0]
    rows = np.nonzero(d.any(axis=(0, 2)))[0]
    print((c, h, w), "r equal:", not d.any(), "ndiff", d.sum(), "rows", rows[:12], "norms", res[0][1], res[2][1], flush=True)
    if d.any():
        ci, yi, xi = np.nonzero(d)
        for k in range(3):
            print("   ", ci[k], yi[k], xi[k], res[0][0][ci[k], yi[k], xi[k]], res[2][0][ci[k], yi[k], xi[k]])
lib.sp_march_variant(2)
