"""Row-strip partitioned solve (csrc/strips.cu) on one GPU:
P logical strips exchange halos through device copies.  The partition is
invisible in the result: every P gives the bit-identical solve, and the
solve agrees with the single-hierarchy solver to solver tolerance."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _inst(c, h, w, density=0.05, seed=0):
    f = O.synth(h, w, c, seed)
    mask = (np.random.default_rng(seed + 7).random((h, w)) < density).astype(np.uint8)
    return f, mask


@pytest.mark.parametrize("shape,Ps", [((3, 1024, 1536), (1, 2, 4)), ((1, 517, 640), (1, 2, 3))])
def test_partition_is_bit_invisible_cold_fmg(shape, Ps):
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver, max_partitioned_levels
    c, h, w = shape
    f, mask = _inst(c, h, w)
    La = min(max_partitioned_levels(h, w, P) for P in Ps)
    assert La >= 1
    cfg = sp.MultigridConfig(tol=1e-6, max_cycles=60)
    outs, reps = [], []
    for P in Ps:
        s = StripSolver(h, w, c, strips=P, cfg=cfg, La=La)
        u, rep = s.inpaint(sp.Image(f), sp.Mask(mask))
        outs.append(u.data)
        reps.append(rep)
    for u, rep in zip(outs[1:], reps[1:]):
        assert np.array_equal(u, outs[0])
        assert rep.iterations == reps[0].iterations
        assert rep.residuals == reps[0].residuals
    assert reps[0].converged and reps[0].residuals[-1] <= 1e-6
    # the single-hierarchy solver to the same tolerance
    ur, repr_ = sp.inpaint(sp.Image(f), sp.Mask(mask), cfg)
    assert repr_.converged
    rel = np.linalg.norm(outs[0] - ur.data) / np.linalg.norm(ur.data)
    assert rel <= 1e-5
    assert np.array_equal(outs[0][:, mask > 0], f.astype(np.float32)[:, mask > 0])


def test_partition_is_bit_invisible_warm_cycles():
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    c, h, w = 3, 768, 1024
    f, mask = _inst(c, h, w, density=0.03, seed=3)
    u0, _ = sp.inpaint(sp.Image(f), sp.Mask(mask), sp.MultigridConfig(tol=1e-2))
    cfg = sp.MultigridConfig(tol=None, cycles=3)
    outs = []
    for P in (1, 2, 4):
        s = StripSolver(h, w, c, strips=P, cfg=cfg, La=2)
        u, rep = s.inpaint(sp.Image(f), sp.Mask(mask), init=u0)
        assert rep.iterations == 3 and rep.converged
        outs.append(u.data)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    ur, _ = sp.inpaint(sp.Image(f), sp.Mask(mask), cfg, init=u0)
    assert np.abs(outs[0] - ur.data).max() <= 1e-3 * np.abs(ur.data).max()


def test_strip_solver_validation():
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver
    with pytest.raises(ValueError):
        StripSolver(256, 256, 1, strips=2, cfg=sp.MultigridConfig(dtype="float64"))
    s = StripSolver(256, 256, 1, strips=2, La=1)
    with pytest.raises(ValueError):
        s.inpaint(sp.Image(np.ones((1, 256, 256))), sp.Mask(np.zeros((256, 256))))


def test_pipeline_on_strips_is_partition_invariant():
    """run_pipeline with every inpainting / B / B^T solve on row strips:
    the same mask and tonal values for every strip count, and the same
    optimisation quality as the single-hierarchy pipeline."""
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200.strips import StripSolver, max_partitioned_levels
    c, h, w = 3, 512, 768
    f = O.synth(h, w, c, 4)
    cfg = sp.PipelineConfig(iterations=6)
    La = min(max_partitioned_levels(h, w, P) for P in (2, 3))
    runs = []
    for P in (1, 2, 3):
        solver = StripSolver(h, w, c, strips=P, cfg=cfg.solver().cfg, La=La)
        mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg, solver=solver)
        runs.append((mask.indicator.copy(), st.g.data.copy(), st.mse, [r[2] for r in hist]))
    for m, g, mse, hh in runs[1:]:
        assert np.array_equal(m, runs[0][0])
        assert np.array_equal(g, runs[0][1])
        assert mse == runs[0][2] and hh == runs[0][3]
    mask_r, st_r, hist_r, _ = sp.run_pipeline(sp.Image(f), cfg)
    assert mask_r.count == int(runs[0][0].sum())
    assert abs(st_r.mse - runs[0][2]) <= 5e-3 * st_r.mse
