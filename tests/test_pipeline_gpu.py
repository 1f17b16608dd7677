"""End-to-end run_pipeline on the GPU vs the reference's recorded runs and
the oracle; the B1 kernel-table monkeypatch path (test_backends.py:132-152
style) driving the oracle orchestration with the CUDA kernels."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
S = json.load(open(os.path.join(HERE, "golden", "reference_scalars.json")))


@pytest.fixture(scope="module")
def sp():
    import paper_2401_06747_b200 as sp
    return sp


@pytest.mark.parametrize("key", ["textured64_dd_none", "textured64_dd_rasvi",
                                 "textured64_dd_vi"])
def test_recorded_reference_runs(sp, textured64, key):
    """pkg/test_output.txt:64-67 (8 printed digits)."""
    rec = S["recorded"][key]
    f = np.clip(np.rint(textured64), 0, 255)
    tonal = {"none": "none", "ras+vi": "ras+vi", "voronoi-init": "voronoi-init"}[rec["tonal"]]
    cfg = sp.PipelineConfig(density=rec["density"], iterations=rec["iterations"],
                            seed=rec["seed"], tonal=tonal)
    mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg)
    assert abs(st.mse - rec["mse"]) <= 1e-4 * rec["mse"]


@pytest.mark.parametrize("h,w,c", [(64, 64, 3), (128, 128, 1), (96, 160, 3)])
def test_pipeline_matches_oracle(sp, h, w, c):
    f = O.synth(h, w, c, 0)
    mask, st, hist, _ = sp.run_pipeline(sp.Image(f), sp.PipelineConfig())
    m2, st2, h2, _ = O.run_pipeline(f)
    assert mask.count == int(m2.sum()) == int(0.05 * h * w)
    # densification is chaotic in the argmax picks (the
    # reference's own two backends differ by ~0.3% in MSE at 256^2); at
    # these sizes the masks agree to a few pixels and the MSE to 0.5%
    assert (mask.indicator != m2).sum() <= 0.05 * m2.sum()
    assert abs(st.mse - st2["mse"]) <= 5e-3 * st2["mse"]


def test_pipeline_outputs_interpolate(sp):
    f = O.synth(48, 64, 3, 1)
    mask, st, _, _ = sp.run_pipeline(sp.Image(f), sp.PipelineConfig(iterations=5))
    m = mask.indicator.astype(bool)
    assert np.array_equal(st.u.data[:, m], st.g.data[:, m])
    assert np.all(st.g.data[:, ~m] == 0)


@pytest.mark.parametrize("spatial", ["aa", "random"])
@pytest.mark.parametrize("tonal", ["none", "balance", "cgnr", "ras"])
def test_other_methods_run(sp, spatial, tonal):
    f = O.synth(40, 40, 1, 2)
    cfg = sp.PipelineConfig(spatial=spatial, tonal=tonal, iterations=4)
    mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg)
    assert mask.count == int(0.05 * 1600)
    assert np.isfinite(st.mse)


def test_ps_baselines_reduce_to_target(sp):
    f = O.synth(24, 24, 1, 3)
    m = sp.probabilistic_sparsify(sp.Image(f), 0.1, sp.PsConfig(seed=1))
    assert m.count == int(0.1 * 576)
    m2 = sp.nlpe(sp.Image(f), m, sp.NlpeConfig(cycles=1, candidates=2))
    assert m2.count == m.count


def test_kernel_table_drives_oracle_orchestration(sp):
    """B1: swap the CUDA kernel table under the oracle orchestration (the
    reference's monkeypatch pattern) -- inpaint agrees with the CPU table."""
    from paper_2401_06747_b200.kernels import cuda_impl
    f = O.synth(37, 29, 3, 8)
    m = (np.random.default_rng(8).random((37, 29)) < 0.15).astype(np.uint8)
    cfg = O.SolverCfg(dtype="float64", tol=1e-8)
    u_cpu, _ = O.inpaint(f, m, cfg)
    saved = {n: getattr(O, n) for n in O.KERNEL_NAMES}
    try:
        for n in O.KERNEL_NAMES:
            setattr(O, n, getattr(cuda_impl, n))
        u_gpu, rep = O.inpaint(f, m, cfg)
    finally:
        for n, fn in saved.items():
            setattr(O, n, fn)
    assert rep.converged
    assert np.linalg.norm(u_gpu - u_cpu) / np.linalg.norm(u_cpu) <= 1e-6
