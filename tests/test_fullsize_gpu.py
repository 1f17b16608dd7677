"""BASELINE.json configs[3] at full size (3840x2160 RGB, 5% density,
PipelineConfig defaults): size-independent properties plus the reference's
own 4K run as recorded by the survey (`dd` MSE
421.8 -> 17.41 with exactly 414,720 stored pixels, `ras+vi` final MSE
14.55; two printed decimals).  Masks of whole runs are not bit-comparable
(the reference's own backends disagree by ~0.3% in MSE), so
the MSEs are checked to 0.5% -- the lockstep bit-exact geometry contract is
tests/test_geometry_gpu.py."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

REF_DD_MSE, REF_FINAL_MSE, REF_COUNT = 17.41, 14.55, 414_720


@pytest.fixture(scope="module")
def run4k():
    import paper_2401_06747_b200 as sp
    f = O.synth(2160, 3840, 3, 0)
    mask, state, hist, _ = sp.run_pipeline(sp.Image(f), sp.PipelineConfig())
    return f, mask, state, hist


def test_4k_pipeline_mask_budget_and_history(run4k):
    f, mask, state, hist = run4k
    assert mask.count == REF_COUNT == int(0.05 * 2160 * 3840)
    mses = [row[2] for row in hist]
    assert abs(mses[0] - 421.8) <= 0.005 * 421.8          # cold FMG on the dithered mask
    assert abs(mses[-1] - REF_DD_MSE) <= 0.005 * REF_DD_MSE
    assert all(b <= a * 1.05 for a, b in zip(mses, mses[1:]))  # densification improves


def test_4k_tonal_optimum(run4k):
    f, mask, state, hist = run4k
    assert abs(state.mse - REF_FINAL_MSE) <= 0.005 * REF_FINAL_MSE
    assert state.mse < hist[-1][2]
    # the reconstruction interpolates the stored values exactly
    m = mask.indicator.astype(bool)
    g, u = state.g.data, state.u.data
    assert np.array_equal(u[:, m], g[:, m])
    assert np.all(g[:, ~m] == 0)
