"""Host-driven vs device-driven (graph WHILE node) tolerance loop on warm 4K
RGB solves: wall time per solve and V-cycles.  `python scripts/probe_loop.py
[switch]` toggles another 0/1 library switch instead (e.g. sp_spec_vcycle)."""
import os, sys, time
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
SWITCH = sys.argv[1] if len(sys.argv) > 1 else "sp_graph_loop"
for gl in (0, 1, 0, 1):
    getattr(lib, SWITCH)(gl)
    _POOL.clear()
    hier = GridHierarchy.build(sp.Mask(mask), sp.Image(f), sp.MultigridConfig(), channels=C)
    u, rep = hier.solve_sym(bsym, tol=1e-4, cascade=True)
    for tol in (1e-4, 1e-6):
        ut = u + 0.5  # a perturbed warm start
        hier.solve_sym(bsym, init=ut, tol=tol)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            u2, rep2 = hier.solve_sym(bsym, init=ut, tol=tol)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5 * 1e3
        print(f"{SWITCH}={gl} tol={tol}: {dt:.3f} ms/solve, {rep2.iterations} V-cycles "
              f"({dt / max(1, rep2.iterations):.3f} ms/cycle)", flush=True)
        # the same number of V-cycles without tolerance tests
        n = rep2.iterations
        hier.solve_sym(bsym, init=ut, tol=None, cycles=n)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            hier.solve_sym(bsym, init=ut, tol=None, cycles=n)
        torch.cuda.synchronize()
        dt2 = (time.perf_counter() - t) / 5 * 1e3
        print(f"{SWITCH}={gl} fixed {n} cycles: {dt2:.3f} ms/solve", flush=True)
