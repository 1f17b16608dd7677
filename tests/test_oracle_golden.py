"""Pin the CPU oracle to the reference: every oracle function against the
fixtures the reference itself produced (tests/golden/make_golden.py, numba
backend, numpy 2.3 / scipy 1.18).  Bit-exact throughout -- the oracle
restates the reference's arithmetic order.  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_vectors.npz"))
S = json.load(open(os.path.join(HERE, "golden", "reference_scalars.json")))


def _inst(dt):
    rng = np.random.default_rng(8)
    x = rng.uniform(0, 255, (3, 37, 29)).astype(dt)
    mask = (rng.random((37, 29)) < 0.15).astype(np.uint8)
    return x, mask


@pytest.mark.parametrize("tag,dt", [("f32", np.float32), ("f64", np.float64)])
def test_kernel_table_bit_exact(tag, dt):
    x, mask = _inst(dt)
    for name in ("inpaint_matvec", "sym_matvec", "sym_rhs", "ct_apply"):
        assert np.array_equal(getattr(O, name)(x, mask, 1.0), G[f"k_{name}_{tag}"]), name
    assert np.array_equal(O.negated_laplacian(x, 1.0), G[f"k_negated_laplacian_{tag}"])
    bs = O.sym_rhs(np.where(mask[None] > 0, x, 0).astype(dt), mask, 1.0)
    r, n = O.sym_residual(x, bs, mask, 1.0)
    assert np.array_equal(r, G[f"k_sym_residual_r_{tag}"])
    assert np.array_equal(n, G[f"k_sym_residual_n_{tag}"])
    assert np.array_equal(O.restrict_values(x), G[f"k_restrict_values_{tag}"])
    cm, cv = O.restrict_mask(mask, x)
    assert np.array_equal(cm, G[f"k_restrict_mask_m_{tag}"])
    assert np.array_equal(cv, G[f"k_restrict_mask_v_{tag}"])
    assert np.array_equal(O.prolongate(O.restrict_values(x), 37, 29), G[f"k_prolongate_{tag}"])
    for blk, ov in ((16, 4), (32, 6)):
        d = O.build_decomposition(37, 29, blk, ov)
        u = np.zeros_like(x)
        m = np.broadcast_to(mask[None].astype(bool), u.shape)
        u[m] = bs[m]
        r0, n0 = O.sym_residual(u, bs, mask, 1.0)
        taus = 0.25 * (d["bh"] * d["bw"] / mask.size) * n0
        O.oras_apply(u, r0, mask, d["xs"], d["ys"], d["bh"], d["bw"], 0.0, taus,
                     d["bh"] * d["bw"], d["weights"].astype(dt), 1.0)
        assert np.array_equal(u, G[f"k_oras_{blk}_{tag}"]), blk


def test_geometry_kernels_bit_exact():
    rng = np.random.default_rng(3)
    pick = np.sort(rng.choice(48 * 48, 30, replace=False))
    seeds = np.stack(np.unravel_index(pick, (48, 48)), axis=1).astype(np.int64)
    lab = np.full((48, 48), -1, np.int32)
    lab[seeds[:, 0], seeds[:, 1]] = np.arange(30, dtype=np.int32)
    labels = O.jfa_run(lab, seeds, np.array([1, 32, 16, 8, 4, 2, 1]))
    assert np.array_equal(labels, G["k_jfa_labels"])
    assert np.array_equal(O.jfa_dist2(labels, seeds), G["k_jfa_dist2"])
    rng = np.random.default_rng(4)
    assert np.array_equal(O.fs_dither(np.clip(rng.uniform(0, 0.4, (40, 33)), 0, 1)),
                          G["k_fs_dither"])
    rng = np.random.default_rng(5)
    vy = rng.integers(0, 40, 12).astype(np.int64)
    vx = rng.integers(0, 40, 12).astype(np.int64)
    tris = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6], [6, 7, 8], [8, 9, 10]], np.int64)
    a = O.assign_triangles(tris, vy, vx, 40, 40)
    assert np.array_equal(a, G["k_assign"])
    err = rng.uniform(0, 1, (40, 40))
    s_, i_, v_ = O.reduce_cells(np.where(a < 0, 0, a).astype(np.int32), err, 5)
    assert np.array_equal(s_, G["k_reduce_sums"]) and np.array_equal(i_, G["k_reduce_amax"])
    assert np.array_equal(v_, G["k_reduce_aval"])


@pytest.mark.parametrize("hh,ww,cc,seed", [(64, 64, 3, 0), (96, 80, 1, 7), (128, 128, 3, 2)])
def test_dithered_initial_mask_bit_exact(hh, ww, cc, seed):
    f = O.synth(hh, ww, cc, seed)
    n = hh * ww
    init, _ = O.schedule(int(0.05 * n), 20)
    m = O.analytic_mask(f, init / n, dither="random", sigma=1.0, seed=seed, count=init)
    assert np.array_equal(m, G[f"initmask_{hh}x{ww}x{cc}_s{seed}"])


def test_textured_masks_bit_exact(textured64):
    assert np.array_equal(O.analytic_mask(textured64, 0.07, dither="random", seed=5),
                          G["initmask_textured64_d007_s5"])
    assert np.array_equal(O.analytic_mask(textured64, 0.05), G["aamask_textured64_d005"])


def test_densify_trace_and_final_mask_bit_exact():
    f = O.synth(64, 64, 3, 0)
    trace = []
    mask, u, hist = O.delaunay_densify(f, 0.05, 10, seed=0, trace=trace)
    for it in (0, 4, 9):
        t = trace[it]
        assert np.array_equal(t["labels"], G[f"dd_it{it}_labels"])
        assert np.array_equal(t["tris"], G[f"dd_it{it}_tris"])
        assert np.array_equal(t["err"], G[f"dd_it{it}_err"])
        assert np.array_equal(t["sums"], G[f"dd_it{it}_sums"])
        assert np.array_equal(t["amax"], G[f"dd_it{it}_amax"])
    assert np.array_equal(mask, G["dd_final_mask"])
    assert [h[2] for h in hist] == S["dd_history_mse"]


def test_tonal_bit_exact():
    f = O.synth(64, 64, 3, 0)
    mask = G["dd_final_mask"]
    vi = O.voronoi_richardson_init(f, mask)
    assert vi["mse"] == S["vi_mse"] and vi["iterations"] == S["vi_steps"]
    ras = O.ras_tonal(f, mask, init=vi)
    assert ras["mse"] == S["ras_mse"] and ras["iterations"] == S["ras_outer"]
    assert np.array_equal(ras["g"].astype(np.float32), G["tonal_ras_g"])
    cg = O.cgnr_tonal(f, mask)
    assert cg["mse"] == S["cgnr_mse"] and cg["iterations"] == S["cgnr_iters"]


def test_inpaint_f64_bit_exact():
    f = O.synth(48, 40, 3, 5)
    m = (np.random.default_rng(9).random((48, 40)) < 0.08).astype(np.uint8)
    u, rep = O.inpaint(f, m, O.SolverCfg(dtype="float64", tol=1e-10, max_cycles=200))
    assert np.array_equal(u, G["inpaint_48x40_u"])
    assert rep.iterations == S["inpaint_48x40_iters"]


@pytest.mark.parametrize("key", ["textured64_dd_none", "textured64_dd_rasvi",
                                 "textured64_dd_vi"])
def test_recorded_reference_runs(textured64, key):
    """The reference's own recorded CLI lines (pkg/test_output.txt:64-67),
    printed with 8 significant digits."""
    rec = S["recorded"][key]
    f = np.clip(np.rint(textured64), 0, 255)  # the PGM the CLI test writes
    cfg = O.SolverCfg()
    mask, _, _ = O.delaunay_densify(f, rec["density"], rec["iterations"], seed=rec["seed"],
                                    cfg=cfg)
    if rec["tonal"] == "none":
        u, _ = O.inpaint(f, mask, cfg, tol=1e-6)
        mse = O.mse(f, u)
    else:
        st = O.voronoi_richardson_init(f, mask, cfg)
        if rec["tonal"] == "ras+vi":
            st = O.ras_tonal(f, mask, init=st, cfg=cfg)
        mse = st["mse"]
    assert abs(mse - rec["mse"]) <= 5e-7 * rec["mse"]


def test_neighbor_balance_oracle_matches_reference():
    """tonal.py:389-414 stored values vs the reference's own output
    (tests/golden/large_f34.npz, scipy.ndimage.correlate)."""
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "large_f34.npz"))
    g = O.neighbor_balance_values(G["t64_pgm"], G["balance_u_in"], G["aa_mask"])
    assert np.array_equal(g, G["balance_g_nosolver"])
