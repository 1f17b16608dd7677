import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200.solver import GridHierarchy, _masked_rhs, _POOL
from oracle import oracle as O
lib = _lib.load()
c, h, w = 1, 128, 128
f = O.synth(h, w, c, 0)
mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
ft = torch.from_numpy(f).float().cuda(); mt = torch.from_numpy(mask).cuda()
u0 = ft.clone()
print("u0 row0", u0[0, 0, :5].tolist(), "row1", u0[0, 1, :3].tolist(), "mask", mask[0, :4], flush=True)
bsym = _masked_rhs(ft, mt)
print("b row0", bsym[0, 0, :3].tolist(), flush=True)
lib.sp_march_variant(2); _POOL.clear()
hier = GridHierarchy.build(sp.Mask(mt), sp.Image(ft), sp.MultigridConfig())
hier.solve_sym(bsym, init=u0, tol=1e9)
r = torch.empty_like(ft); nrm = torch.empty(c, dtype=torch.float64, device="cuda")
_lib.call("sp_hier_residual", hier._h, 0, _lib.ptr(r), _lib.ptr(nrm), _lib.stream())
torch.cuda.synchronize()
print("r row0", r[0, 0, :4].tolist())
