"""A/B of the warp-streamed vs CTA-tile TMA sweeps on the 4K RGB hierarchy:
per-kernel CUDA-event times (sp_hier_bench) and the warm V-cycle time."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import _lib
from paper_2401_06747_b200.solver import GridHierarchy, _masked_rhs, _POOL
from oracle import oracle as O

H, W, C = 2160, 3840, 3
lib = _lib.load()
f = torch.from_numpy(O.synth(H, W, C, 0)).float().cuda()
mask = (torch.from_numpy(np.random.default_rng(2).random((H, W)) < 0.05)).to(torch.uint8).cuda()
bsym = _masked_rhs(f, mask)
names = {0: "resid", 1: "oras", 2: "blend", 3: "resid+restrict", 4: "prolong"}
# ws:prefetch:stages[:oras_offbits[:blend_packed]]
variants = [tuple(map(int, a.split(":"))) for a in sys.argv[1:]] or [(0, 0, 2), (1, 2, 2)]
for var in variants:
    ws, pf, spw = var[:3]
    ob = var[3] if len(var) > 3 else 1
    bp = var[4] if len(var) > 4 else 1
    lib.sp_oras_offbits(ob)
    lib.sp_blend_packed(bp)
    lib.sp_ws_variant(ws)
    lib.sp_ws_prefetch(pf)
    lib.sp_ws_stages(spw)
    _POOL.clear()
    hier = GridHierarchy.build(sp.Mask(mask), sp.Image(f), sp.MultigridConfig(), channels=C)
    u, rep = hier.solve_sym(bsym, tol=1e-4, cascade=True)
    out = []
    for which in (0, 3, 4, 2, 1):
        t_ms, nb = ctypes.c_double(), ctypes.c_double()
        _lib.call("sp_hier_bench", hier._h, which, 20, ctypes.byref(t_ms), ctypes.byref(nb),
                  _lib.stream())
        out.append(f"{names[which]} {t_ms.value*1e3:.1f} us ({nb.value/t_ms.value/1e6:.0f} GB/s)")
    hier.solve_sym(bsym, init=u, tol=None, cycles=2)
    torch.cuda.synchronize()
    t = time.perf_counter()
    hier.solve_sym(bsym, init=u, tol=None, cycles=20)
    torch.cuda.synchronize()
    vc = (time.perf_counter() - t) / 20 * 1e3
    print(f"ws={ws} pf={pf} spw={spw} offbits={ob} bpack={bp}: V-cycle {vc:.3f} ms | " + " | ".join(out), flush=True)
