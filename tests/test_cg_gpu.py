"""`cg_solve` (solver.py:422-482) on the device: the reference's own
TestCgSolve cases (test_solver.py:13-45), with the operator given in the
caller's representation (numpy for an array rhs, Image for an Image rhs),
plus the hierarchy shape guards (a hierarchy built for C channels refuses a
rhs of another channel count instead of reading out of bounds)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import paper_2401_06747_b200 as sp
    return sp


def test_identity_converges_in_one_iteration(sp, rng):
    rhs = sp.Image(rng.uniform(0, 1, (1, 6, 6)))
    out, rep = sp.cg_solve(lambda x: x, rhs, tol=1e-12)
    assert rep.iterations == 1 and rep.converged
    assert np.allclose(out.data, rhs.data)


def test_exact_init_takes_zero_iterations(sp, rng):
    rhs = sp.Image(rng.uniform(0, 1, (1, 6, 6)))
    out, rep = sp.cg_solve(lambda x: x, rhs, init=rhs.copy(), tol=1e-12)
    assert rep.iterations == 0 and rep.converged


def _dense_sym(mask):
    n = mask.size
    a = np.empty((n, n))
    for j in range(n):
        e = np.zeros((1,) + mask.shape)
        e.ravel()[j] = 1.0
        a[:, j] = O.sym_matvec(e, mask, 1.0).ravel()
    return a


def test_matches_dense_solve_on_symmetrized_system(sp, rng):
    """test_solver.py:26-39: a numpy operator; the result is numpy."""
    f = rng.uniform(0, 255, (1, 8, 8))
    mask = (rng.random((8, 8)) < 0.25).astype(np.uint8)
    mask[0, 0] = 1
    a = _dense_sym(mask)
    b = O.sym_rhs(np.where(mask[None] > 0, f, 0.0), mask, 1.0)
    want = np.linalg.solve(a, b[0].ravel())
    seen = []

    def op(x):
        seen.append(type(x))
        return O.sym_matvec(x, mask, 1.0)

    got, rep = sp.cg_solve(op, b, tol=1e-10)
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    assert all(t is np.ndarray for t in seen)
    assert rep.converged
    assert np.linalg.norm(got[0].ravel() - want) / np.linalg.norm(want) <= 1e-8
    # the oracle's CG trace (same recurrences, double dots)
    assert rep.iterations <= 64


def test_breakdown_is_reported(sp):
    out, rep = sp.cg_solve(lambda x: -x, np.ones((1, 2, 2)), tol=1e-12, max_iters=10)
    assert rep.breakdown and isinstance(out, np.ndarray)


def test_device_tensor_rhs_stays_on_device(sp):
    import torch
    b = torch.ones((1, 4, 4), dtype=torch.float64, device="cuda")
    out, rep = sp.cg_solve(lambda x: 2.0 * x, b, tol=1e-12)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert torch.allclose(out, b / 2)


def test_hierarchy_rejects_channel_mismatch(sp, rng):
    import torch
    m = (rng.random((40, 40)) < 0.1).astype(np.uint8)
    m[0, 0] = 1
    hier = sp.InpaintSolver().hierarchy(sp.Mask(m))            # 1 channel
    rgb = torch.zeros((3, 40, 40), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        hier.solve_sym(rgb)
    with pytest.raises(ValueError):
        hier.vcycle_inplace(rgb, rgb)
    u, rep = hier.solve_sym(rgb[:1].contiguous(), tol=1e-4)
    assert u.shape == (1, 40, 40)


def test_vcycle_rebuilds_for_other_channel_count(sp):
    f = O.synth(40, 48, 3, 1)
    m = (np.random.default_rng(3).random((40, 48)) < 0.1).astype(np.uint8)
    solver = sp.InpaintSolver()
    hier = solver.hierarchy(sp.Mask(m))                        # 1 channel
    u0 = sp.Image(np.zeros_like(f))
    out = sp.vcycle(u0, sp.Image(f), sp.Mask(m), hier)
    assert out.data.shape == f.shape
    # every channel got a real V-cycle (nothing left uninitialised)
    ref = sp.vcycle(sp.Image(np.zeros_like(f[:1])), sp.Image(f[:1]), sp.Mask(m), hier)
    assert np.array_equal(out.data[0], ref.data[0])


def test_handle_pool_is_bounded(sp):
    from paper_2401_06747_b200.solver import _POOL
    for k in range(10):
        h = 24 + 8 * k
        m = np.zeros((h, h), np.uint8)
        m[1, 1] = 1
        sp.inpaint(sp.Image(np.ones((1, h, h))), sp.Mask(m))
    assert len(_POOL) <= _POOL.max_total
