"""Device-resident multigrid solver (B2) vs the CPU oracle."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _cfg(dtype, tol):
    from paper_2401_06747_b200 import MultigridConfig
    return MultigridConfig(dtype=dtype, tol=tol, max_cycles=200)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("shape,density", [((1, 64, 64), 0.1), ((3, 37, 53), 0.08),
                                           ((1, 256, 256), 0.1)])
def test_inpaint_matches_oracle(dtype, shape, density):
    import paper_2401_06747_b200 as sp
    f = O.synth(shape[1], shape[2], shape[0], 0)
    mask = (np.random.default_rng(1).random(shape[1:]) < density).astype(np.uint8)
    tol = 1e-6 if dtype == "float32" else 1e-10
    u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), _cfg(dtype, tol))
    uo, repo = O.inpaint(f, mask, O.SolverCfg(dtype=dtype, tol=tol, max_cycles=200))
    assert rep.converged
    assert rep.residuals[-1] <= tol
    # the relative residual recomputed by the oracle (numba_impl.py:147-158
    # arithmetic, f64 norms) on the returned u, not the solver's own partials
    fd = f.astype(dtype)
    bsym = O.sym_rhs(np.where(mask[None] > 0, fd, 0).astype(dtype), mask, 1.0)
    _, norms = O.sym_residual(np.ascontiguousarray(u.data, dtype), bsym, mask, 1.0)
    rres = np.sqrt(norms.sum()) / np.linalg.norm(bsym.astype(np.float64))
    assert rres <= tol * 1.01
    rel = np.linalg.norm(u.data - uo) / np.linalg.norm(uo)
    assert rel <= (1e-4 if dtype == "float32" else 1e-8)
    assert np.array_equal(u.data[:, mask > 0], f.astype(u.data.dtype)[:, mask > 0])


def test_inpaint_default_tol_tracks_oracle_iterations():
    import paper_2401_06747_b200 as sp
    f = O.synth(256, 256, 1, 0)
    mask = (np.random.default_rng(1).random((256, 256)) < 0.10).astype(np.uint8)
    u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask))
    uo, repo = O.inpaint(f, mask)
    assert abs(rep.iterations - repo.iterations) <= 1
    rel = np.linalg.norm(u.data - uo) / np.linalg.norm(uo)
    assert rel <= 1e-3


def test_warm_start_and_fixed_cycles():
    import paper_2401_06747_b200 as sp
    f = O.synth(96, 80, 3, 2)
    mask = (np.random.default_rng(5).random((96, 80)) < 0.05).astype(np.uint8)
    u0, _ = sp.inpaint(sp.Image(f), sp.Mask(mask))
    uo0, _ = O.inpaint(f, mask)
    cfg = sp.MultigridConfig(tol=None, cycles=2)
    u1, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), cfg, init=u0)
    uo1, _ = O.inpaint(f, mask, O.SolverCfg(tol=None, cycles=2), init=uo0)
    assert rep.iterations == 2 and rep.converged
    assert np.linalg.norm(u1.data - uo1) / np.linalg.norm(uo1) <= 1e-4


def test_empty_mask_raises():
    import paper_2401_06747_b200 as sp
    with pytest.raises(ValueError):
        sp.inpaint(sp.Image(np.ones((1, 8, 8))), sp.Mask(np.zeros((8, 8))))


@pytest.mark.parametrize("shape", [(3, 301, 512), (1, 260, 384)])
def test_sweep_kernel_variants_agree(shape):
    """The TMA-staged (mgtma.cu) and row-marching (mgfast.cu) sweeps of the
    wide float levels use the reference arithmetic of mg.cu's per-pixel
    kernels: the same V-cycles from the same start agree to the last bits
    (only the norm summation order differs)."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 3)
    mask = (np.random.default_rng(4).random((h, w)) < 0.05).astype(np.uint8)
    outs = []
    prev, prev_ws = lib.sp_march_variant(-1), lib.sp_ws_variant(-1)
    prev_px = lib.sp_tma_min_pixels(-1)
    lib.sp_tma_min_pixels(0)  # the TMA kernels on every level that fits them
    try:
        # (sweep variant, warp-streamed TMA kernels on/off)
        for mv, ws in ((2, 1), (2, 0), (1, 1), (0, 1)):
            lib.sp_march_variant(mv)
            lib.sp_ws_variant(ws)
            _POOL.clear()
            u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=None, cycles=3))
            outs.append(u.data)
    finally:
        lib.sp_march_variant(prev)
        lib.sp_ws_variant(prev_ws)
        lib.sp_tma_min_pixels(prev_px)
        _POOL.clear()
    for o in outs[:3]:
        rel = np.abs(o - outs[3]).max() / np.abs(outs[3]).max()
        assert rel <= 1e-6


@pytest.mark.parametrize("shape", [(1, 128, 128), (1, 200, 256), (3, 130, 384), (3, 67, 512),
                                   (1, 75, 272)])
def test_sweep_kernel_residuals_bit_identical(shape):
    """The residual r = b~ - A~ u of one iterate computed by the TMA-staged,
    row-marching and per-pixel sweep kernels: bit-identical (numba_impl.py
    147-158 arithmetic in all three); norms equal to summation order."""
    import torch
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import GridHierarchy, _POOL, _masked_rhs
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 0)
    mask = (np.random.default_rng(7).random((h, w)) < 0.05).astype(np.uint8)
    ft = torch.from_numpy(f).float().cuda()
    mt = torch.from_numpy(mask).cuda()
    u0 = ft + torch.from_numpy(np.random.default_rng(8).standard_normal(f.shape)).float().cuda()
    bsym = _masked_rhs(ft, mt)
    prev, prev_ws = lib.sp_march_variant(-1), lib.sp_ws_variant(-1)
    prev_px = lib.sp_tma_min_pixels(-1)
    lib.sp_tma_min_pixels(0)  # the TMA kernels on every level that fits them
    res = {}
    try:
        # 3: the CTA-tile TMA kernels (sweep 2 with the warp-streamed off)
        for v in (0, 1, 2, 3):
            lib.sp_march_variant(min(v, 2))
            lib.sp_ws_variant(0 if v == 3 else 1)
            _POOL.clear()
            hier = GridHierarchy.build(sp.Mask(mt), sp.Image(ft), sp.MultigridConfig())
            hier.solve_sym(bsym, init=u0, tol=1e9)      # u = u0 (enforced), no cycle
            r = torch.empty_like(ft)
            nrm = torch.empty(c, dtype=torch.float64, device="cuda")
            _lib.call("sp_hier_residual", hier._h, 0, _lib.ptr(r), _lib.ptr(nrm), _lib.stream())
            res[v] = (r.cpu().numpy(), nrm.cpu().numpy())
    finally:
        lib.sp_march_variant(prev)
        lib.sp_ws_variant(prev_ws)
        lib.sp_tma_min_pixels(prev_px)
        _POOL.clear()
    for v in (1, 2, 3):
        assert np.array_equal(res[v][0], res[0][0])
        assert np.allclose(res[v][1], res[0][1], rtol=1e-6, atol=0)


def _with_oras_variant(v, fn):
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    prev = lib.sp_oras_variant(-1)
    try:
        lib.sp_oras_variant(v)
        _POOL.clear()
        return fn()
    finally:
        lib.sp_oras_variant(prev)
        _POOL.clear()


@pytest.mark.parametrize("shape", [(3, 301, 512), (1, 100, 150), (3, 40, 70)])
def test_oras_warp_kernel_bit_identical(shape):
    """One-warp-per-job ORAS local CG (k_oras_warp, variant 4) vs the 4-warp
    k_oras_rows (variant 0): same fused operations, same 8-row dot groups
    and butterfly pairings, so the V-cycles agree bitwise -- on full 32-row
    blocks and on the short blocks of small / coarse levels."""
    import paper_2401_06747_b200 as sp
    c, h, w = shape
    f = O.synth(h, w, c, 3)
    mask = (np.random.default_rng(4).random((h, w)) < 0.05).astype(np.uint8)

    def run():
        u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=None, cycles=3))
        return u.data

    a, b, c = _with_oras_variant(0, run), _with_oras_variant(4, run), _with_oras_variant(6, run)
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("shape", [(3, 301, 512), (1, 100, 150), (3, 40, 70)])
def test_oras_offbits_bit_identical(shape):
    """The default ORAS job reads its row-mask word precomputed with the mask
    pyramid (k_offbits) instead of loading its 32 mask bytes: identical
    V-cycles, on full and on short / narrow blocks, and in the batched RAS
    block solves."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 3)
    mask = (np.random.default_rng(4).random((h, w)) < 0.05).astype(np.uint8)
    outs = []
    prev = lib.sp_oras_offbits(-1)
    try:
        for v in (1, 0):
            lib.sp_oras_offbits(v)
            _POOL.clear()
            u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=None, cycles=3))
            st = sp.ras_tonal(sp.Image(f), sp.Mask(mask))
            outs.append((u.data, st.g.data, st.mse))
    finally:
        lib.sp_oras_offbits(prev)
        _POOL.clear()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2]


def test_oras_warp_kernel_bit_identical_ras():
    """Batched-tile path (RAS local normal equations, ntile > 1)."""
    import paper_2401_06747_b200 as sp
    f = O.synth(128, 160, 3, 1)
    mask = (np.random.default_rng(2).random((128, 160)) < 0.05).astype(np.uint8)

    def run():
        st = sp.ras_tonal(sp.Image(f), sp.Mask(mask))
        return st.g.data, st.mse

    (ga, ma), (gb, mb) = _with_oras_variant(0, run), _with_oras_variant(4, run)
    assert ma == mb
    assert np.array_equal(ga, gb)


@pytest.mark.parametrize("variant", [7, 8])
@pytest.mark.parametrize("shape", [(3, 301, 512), (1, 100, 150), (3, 2160 // 4, 3840 // 4)])
def test_lean_oras_cg_tracks_reference_ordered_cg(shape, variant):
    """The lean local CG (variant 7: float dots, q = p, fast division;
    variant 8: the same on packed float pairs, FFMA2) against the
    reference-ordered one (variant 6): the same CG iterates up to float
    rounding, so fixed V-cycles agree to ~1e-6 and a tight solve lands on
    the same solution (the oracle-pinned tests run the default)."""
    import paper_2401_06747_b200 as sp
    c, h, w = shape
    f = O.synth(h, w, c, 3)
    mask = (np.random.default_rng(4).random((h, w)) < 0.05).astype(np.uint8)

    def run(cfg):
        return lambda: sp.inpaint(sp.Image(f), sp.Mask(mask), cfg)

    fixed = sp.MultigridConfig(tol=None, cycles=3)
    a = _with_oras_variant(6, run(fixed))[0].data
    b = _with_oras_variant(variant, run(fixed))[0].data
    assert np.linalg.norm(a - b) / np.linalg.norm(a) <= 2e-5
    tight = sp.MultigridConfig(tol=1e-6, max_cycles=200)
    (ua, ra) = _with_oras_variant(6, run(tight))
    (ub, rb) = _with_oras_variant(variant, run(tight))
    assert abs(ra.iterations - rb.iterations) <= 1
    assert np.linalg.norm(ua.data - ub.data) / np.linalg.norm(ua.data) <= 1e-5



@pytest.mark.parametrize("shape", [(3, 301, 512), (3, 2160 // 4, 3840 // 4), (2, 100, 150)])
def test_channel_parallel_vcycle_bit_identical(shape):
    """V-cycle graphs with the C channels as parallel branches on one-channel
    views (solver.cu run_vcycle) vs one sequential chain: bitwise equal."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 5)
    mask = (np.random.default_rng(6).random((h, w)) < 0.05).astype(np.uint8)
    prev = lib.sp_channel_parallel(-1)
    outs = []
    try:
        for on in (0, 1):
            lib.sp_channel_parallel(on)
            _POOL.clear()
            u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=1e-6))
            outs.append((u.data, rep.iterations, rep.residuals))
    finally:
        lib.sp_channel_parallel(prev)
        _POOL.clear()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]


@pytest.mark.parametrize("shape,tol", [((3, 301, 512), 1e-6), ((1, 256, 256), 1e-4),
                                       ((3, 540, 960), 1e-4)])
def test_device_driven_solve_loop_identical(shape, tol):
    """Tolerance solves as one graph launch (WHILE / IF conditional nodes,
    stop test on the device) vs the host-driven loop: same iterate, same
    V-cycle count, same relative-residual history; and the cycle cap."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 7)
    mask = (np.random.default_rng(8).random((h, w)) < 0.05).astype(np.uint8)
    prev = lib.sp_graph_loop(-1)
    outs = []
    try:
        for on in (0, 1):
            lib.sp_graph_loop(on)
            _POOL.clear()
            u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=tol))
            u2, rep2 = sp.inpaint(sp.Image(f), sp.Mask(mask),
                                  sp.MultigridConfig(tol=1e-12, max_cycles=2), init=u)
            outs.append((u.data, rep.iterations, rep.residuals, rep.converged,
                         u2.data, rep2.iterations, rep2.converged))
    finally:
        lib.sp_graph_loop(prev)
        _POOL.clear()
    a, b = outs
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[4], b[4])
    assert a[1:4] == b[1:4] and a[5:] == b[5:]
    assert b[5] == 2 and not b[6]



@pytest.mark.parametrize("shape", [(3, 301, 512), (3, 60, 516), (3, 540, 960), (3, 67, 1300),
                                   (3, 61, 515), (3, 64, 64)])
def test_blend_packed_cover_words_bit_identical(shape):
    """The C = 3 blend with packed per-row / per-column cover words
    (k_oras_blend3p) vs the cover-table chains (k_oras_blend3): the same
    corrections added in the same block order (numba_impl.py:255-263), so
    V-cycles from the same start are bit-identical -- incl. the rows of a
    pulled-in last block with three covers, (3, 60, 516), on the generic
    path; and the column-pair kernel (k_oras_blend3q, mode 2: two pixels per
    8-byte access where W and every block start are even; odd widths keep
    the per-pixel kernel)."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 5)
    mask = (np.random.default_rng(6).random((h, w)) < 0.05).astype(np.uint8)
    outs = []
    prev = lib.sp_blend_packed(-1)
    try:
        for v in (1, 0, 2, 3):
            lib.sp_blend_packed(v)
            _POOL.clear()
            u, rep = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=None, cycles=3))
            outs.append(u.data)
    finally:
        lib.sp_blend_packed(prev)
        _POOL.clear()
    assert np.array_equal(outs[0], outs[1])
    for o in outs[2:]:
        assert np.array_equal(outs[0], o)
