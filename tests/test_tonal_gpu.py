"""Tonal optimization on the GPU vs the oracle / reference fixtures
(north_star tolerance: MSE within 1e-4 relative of the reference's) and the
reference's own tonal unit tests (test_tonal.py)."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_vectors.npz"))
S = json.load(open(os.path.join(HERE, "golden", "reference_scalars.json")))
REL = 1e-4


@pytest.fixture(scope="module")
def sp():
    import paper_2401_06747_b200 as sp
    return sp


def test_vi_ras_cgnr_match_reference(sp):
    f = O.synth(64, 64, 3, 0)
    mask = sp.Mask(G["dd_final_mask"])
    img = sp.Image(f)
    vi = sp.voronoi_richardson_init(img, mask)
    assert vi.iterations == S["vi_steps"]
    assert abs(vi.mse - S["vi_mse"]) <= REL * S["vi_mse"]
    ras = sp.ras_tonal(img, mask, init=vi)
    assert ras.iterations == S["ras_outer"]
    assert abs(ras.mse - S["ras_mse"]) <= REL * S["ras_mse"]
    cg = sp.cgnr_tonal(img, mask)
    assert abs(cg.mse - S["cgnr_mse"]) <= REL * S["cgnr_mse"]
    g = ras.g.data.astype(np.float32)
    on = G["dd_final_mask"].astype(bool)
    assert np.allclose(g[:, on], G["tonal_ras_g"][:, on], rtol=0, atol=1e-2)


@pytest.mark.parametrize("shape,density,seed", [((1, 256, 256), 0.05, 2), ((3, 96, 130), 0.03, 5),
                                                ((1, 70, 200), 0.02, 9)])
def test_tonal_matches_oracle_on_random_masks(sp, shape, density, seed):
    c, h, w = shape
    f = O.synth(h, w, c, seed)
    m = (np.random.default_rng(seed).random((h, w)) < density).astype(np.uint8)
    vi = sp.voronoi_richardson_init(sp.Image(f), sp.Mask(m))
    vo = O.voronoi_richardson_init(f, m)
    assert vi.iterations == vo["iterations"]
    assert abs(vi.mse - vo["mse"]) <= REL * vo["mse"]
    ras = sp.ras_tonal(sp.Image(f), sp.Mask(m), init=vi)
    ro = O.ras_tonal(f, m, init=vo)
    assert abs(ras.mse - ro["mse"]) <= REL * ro["mse"]
    assert ras.mse <= ro["mse"] * (1 + REL)


def test_full_mask_is_identity(sp, rng):
    solver = sp.InpaintSolver(sp.MultigridConfig(dtype="float64"))
    f = sp.Image(rng.uniform(0, 255, (1, 8, 8)))
    full = sp.Mask(np.ones((8, 8)))
    assert np.allclose(sp.apply_B(f, full, solver).data, f.data, atol=1e-8)
    assert np.allclose(sp.apply_Bt(f, full, solver).data, f.data, atol=1e-8)


def test_adjoint_identity(sp, rng):
    """test_tonal.py:42-51: <B x, y> == <x, B^T y>."""
    solver = sp.InpaintSolver(sp.MultigridConfig(dtype="float64"))
    m = rng.random((16, 16)) < 0.1
    m[3, 4] = True
    mask = sp.Mask(m)
    x = sp.Image(rng.standard_normal((1, 16, 16)))
    y = sp.Image(rng.standard_normal((1, 16, 16)))
    bx = sp.apply_B(x, mask, solver, inner_tol=1e-12).data
    bty = sp.apply_Bt(y, mask, solver, inner_tol=1e-12).data
    lhs, rhs = float((bx * y.data).sum()), float((x.data * bty).sum())
    assert abs(lhs - rhs) <= 1e-6 * np.linalg.norm(x.data) * np.linalg.norm(y.data)
    assert np.all(bty[0][~m] == 0.0)


def test_single_pixel_extends_constant(sp):
    solver = sp.InpaintSolver(sp.MultigridConfig(dtype="float64"))
    mask = np.zeros((10, 10))
    mask[4, 6] = 1
    x = np.zeros((1, 10, 10))
    x[0, 4, 6] = 33.0
    out = sp.apply_B(sp.Image(x), sp.Mask(mask), solver, inner_tol=1e-12)
    assert np.allclose(out.data, 33.0, atol=1e-8)


def test_dense_oracle_optimality(sp, rng):
    """test_tonal.py:85-92 and 116-122: CGNR reaches the dense optimum."""
    solver = sp.InpaintSolver(sp.MultigridConfig(dtype="float64"))
    f = sp.Image(rng.uniform(0, 255, (1, 24, 24)))
    m = np.zeros(24 * 24, bool)
    m[rng.choice(24 * 24, 20, replace=False)] = True
    mask = sp.Mask(m.reshape(24, 24))
    want = sp.dense_tonal_oracle(f, mask)
    st = sp.cgnr_tonal(f, mask, solver=solver, rel_improvement=1e-6, max_iters=200,
                       inner_tol=1e-8, final_tol=1e-10)
    assert st.mse <= want.mse * 1.001
    assert st.mse >= want.mse * (1 - 1e-6)


def test_ras_matches_dense_oracle(sp, rng):
    """test_tonal.py:152-159: RAS within 0.1% of the dense optimum."""
    solver = sp.InpaintSolver(sp.MultigridConfig(dtype="float64"))
    f = sp.Image(rng.uniform(0, 255, (1, 40, 40)))
    m = np.zeros(1600, bool)
    m[rng.choice(1600, 60, replace=False)] = True
    mask = sp.Mask(m.reshape(40, 40))
    want = sp.dense_tonal_oracle(f, mask)
    st = sp.ras_tonal(f, mask, cfg=sp.RasTonalConfig(block=16, overlap=4, rel_improvement=1e-6,
                                                      max_outer=200, local_iters=100,
                                                      local_tol=1e-6, inner_tol=1e-8),
                      solver=solver)
    assert st.mse <= want.mse * 1.001


def test_initial_state_and_balance(sp, rng):
    f = O.synth(40, 48, 1, 3)
    m = (rng.random((40, 48)) < 0.1).astype(np.uint8)
    st = sp.initial_state(sp.Image(f), sp.Mask(m))
    u, _ = O.inpaint(f, m, tol=1e-6)
    assert abs(st.mse - O.mse(f, u)) <= 1e-4 * O.mse(f, u)
    bal = sp.neighbor_balance_init(sp.Image(f), st.u, sp.Mask(m))
    assert np.all(bal.g.data[:, m == 0] == 0)


def test_empty_mask_rejected(sp):
    with pytest.raises(ValueError):
        sp.ras_tonal(sp.Image(np.ones((1, 8, 8))), sp.Mask(np.zeros((8, 8))))


def _with_tile_fused(on, fn):
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    prev = lib.sp_tile_fused(-1)
    try:
        lib.sp_tile_fused(on)
        _POOL.clear()
        return fn()
    finally:
        lib.sp_tile_fused(prev)
        _POOL.clear()


@pytest.mark.parametrize("shape,density", [((3, 200, 260), 0.05), ((1, 130, 100), 0.08),
                                           ((3, 64, 64), 0.05), ((2, 90, 50), 0.04)])
def test_fused_tile_solver_matches_batched(sp, shape, density):
    """RAS block-local products on the fused on-chip tile solver (tilesolve.cu,
    one cluster per block) vs the batched V-cycle hierarchy: the same
    element operations, norms summed in another order -> equal to rounding;
    the V-cycle counts per block agree."""
    import torch
    from paper_2401_06747_b200 import tonal
    c, h, w = shape
    f = O.synth(h, w, c, 4)
    mask = (np.random.default_rng(9).random((h, w)) < density).astype(np.uint8)

    def run():
        solver = sp.InpaintSolver()
        blocks = tonal._RasBlocks(torch.from_numpy(mask).cuda(), solver, c, sp.RasTonalConfig())
        rng = np.random.default_rng(3)
        x = torch.from_numpy(rng.standard_normal((blocks.nt, c, blocks.bh, blocks.bw))
                             ).float().cuda()
        act = np.ones(blocks.nt, np.int32)
        act[::3] = 0 if blocks.nt > 2 else 1
        act_d = torch.from_numpy(act).cuda()
        bp = blocks.apply_B(x, act, act_d)
        it = blocks._iters.copy()
        mp = blocks.apply_Bt(bp, act, act_d)
        keep = torch.from_numpy(act > 0).cuda()
        return bp[keep].cpu().numpy(), mp[keep].cpu().numpy(), it[act > 0]

    b1, m1, i1 = _with_tile_fused(1, run)
    b0, m0, i0 = _with_tile_fused(0, run)
    assert np.array_equal(i1, i0)
    for a, b in ((b1, b0), (m1, m0)):
        scale = np.abs(b).max()
        assert np.abs(a - b).max() <= 2e-5 * scale


def test_fused_tile_solver_ras_mse(sp):
    """ras_tonal end to end with and without the fused tile solver."""
    f = O.synth(160, 200, 3, 1)
    mask = (np.random.default_rng(2).random((160, 200)) < 0.05).astype(np.uint8)

    def run():
        st = sp.ras_tonal(sp.Image(f), sp.Mask(mask))
        return st.mse, st.iterations

    (ma, ia), (mb, ib) = _with_tile_fused(1, run), _with_tile_fused(0, run)
    assert ia == ib
    assert abs(ma - mb) <= 1e-6 * mb


@pytest.mark.parametrize("shape", [(3, 256, 320), (1, 300, 200)])
def test_ras_tile_list_bit_identical(shape):
    """The fused RAS block solves of a partly active batch (the tail of the
    local CG) launch over the list of active blocks instead of every block
    with early exits: the same blocks run the same kernels, so ras_tonal is
    bit-identical either way (tonal.py:267-294)."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import _POOL
    lib = _lib.load()
    c, h, w = shape
    f = O.synth(h, w, c, 7)
    mask = (np.random.default_rng(8).random((h, w)) < 0.05).astype(np.uint8)
    outs = []
    prev = lib.sp_tile_list(-1)
    try:
        for v in (1, 0):
            lib.sp_tile_list(v)
            _POOL.clear()
            st = sp.ras_tonal(sp.Image(f), sp.Mask(mask))
            outs.append((st.g.data, st.mse, st.iterations))
    finally:
        lib.sp_tile_list(prev)
        _POOL.clear()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]
