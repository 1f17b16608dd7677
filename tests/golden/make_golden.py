"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/reference_vectors.npz and reference_scalars.json.  The
reference's default backend (numba, kernels/__init__.py:43-66) produces
every array; inputs are deterministic (seeded numpy / the SURVEY.md 8d
`synth` generator), so the tests regenerate the inputs and compare.
Nothing on the GPU box reads /root/reference: the fixtures travel instead.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sparsepaint as sp  # noqa: E402
from sparsepaint import kernels as K  # noqa: E402
from sparsepaint.geometry import (accumulate_errors, delaunay_from_voronoi,  # noqa: E402
                                  jump_flood_voronoi)
from sparsepaint.spatial import _schedule  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import synth  # noqa: E402  (input generator only)


def kernel_instance(dtype):
    rng = np.random.default_rng(8)
    x = rng.uniform(0, 255, (3, 37, 29)).astype(dtype)
    mask = (rng.random((37, 29)) < 0.15).astype(np.uint8)
    return x, mask


def textured64():
    yy, xx = np.mgrid[0:64, 0:64].astype(np.float64)
    return 128 + 60 * np.sin(xx / 5) * np.cos(yy / 7) + 40 * (xx > 40) - 30 * (yy > 50)


def main():
    out = {}
    sc = {"backend": K.BACKEND, "numpy": np.__version__}
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        x, mask = kernel_instance(dt)
        for name in ("inpaint_matvec", "sym_matvec", "sym_rhs", "ct_apply"):
            out[f"k_{name}_{tag}"] = getattr(K, name)(x, mask, 1.0)
        out[f"k_negated_laplacian_{tag}"] = K.negated_laplacian(x, 1.0)
        bs = K.sym_rhs(np.where(mask[None] > 0, x, 0).astype(dt), mask, 1.0)
        r, norms = K.sym_residual(x, bs, mask, 1.0)
        out[f"k_sym_residual_r_{tag}"], out[f"k_sym_residual_n_{tag}"] = r, norms
        out[f"k_restrict_values_{tag}"] = K.restrict_values(x)
        cm, cv = K.restrict_mask(mask, x)
        out[f"k_restrict_mask_m_{tag}"], out[f"k_restrict_mask_v_{tag}"] = cm, cv
        out[f"k_prolongate_{tag}"] = K.prolongate(K.restrict_values(x), 37, 29)
        for blk, ov in ((16, 4), (32, 6)):
            d = sp.build_decomposition(37, 29, blk, ov)
            u = np.zeros_like(x)
            m = np.broadcast_to(mask[None].astype(bool), u.shape)
            u[m] = bs[m]
            r0, n0 = K.sym_residual(u, bs, mask, 1.0)
            taus = 0.25 * (d.bh * d.bw / mask.size) * n0
            K.oras_apply(u, r0, mask, d.xs, d.ys, d.bh, d.bw, 0.0, taus, d.bh * d.bw,
                         d.weights.astype(dt), 1.0)
            out[f"k_oras_{blk}_{tag}"] = u
    # geometry kernels
    rng = np.random.default_rng(3)
    h = w = 48
    pick = np.sort(rng.choice(h * w, 30, replace=False))
    seeds = np.stack(np.unravel_index(pick, (h, w)), axis=1).astype(np.int64)
    lab = np.full((h, w), -1, np.int32)
    lab[seeds[:, 0], seeds[:, 1]] = np.arange(30, dtype=np.int32)
    steps = np.array([1, 32, 16, 8, 4, 2, 1], np.int64)
    out["k_jfa_labels"] = K.jfa_run(lab, seeds, steps)
    out["k_jfa_dist2"] = K.jfa_dist2(out["k_jfa_labels"], seeds)
    rng = np.random.default_rng(4)
    dens = np.clip(rng.uniform(0, 0.4, (40, 33)), 0, 1)
    out["k_fs_dither"] = K.fs_dither(dens)
    rng = np.random.default_rng(5)
    vy = rng.integers(0, 40, 12).astype(np.int64)
    vx = rng.integers(0, 40, 12).astype(np.int64)
    tris = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6], [6, 7, 8], [8, 9, 10]], np.int64)
    a = K.assign_triangles(tris, vy, vx, 40, 40)
    out["k_assign"] = a
    err = rng.uniform(0, 1, (40, 40))
    s_, i_, v_ = K.reduce_cells(np.where(a < 0, 0, a).astype(np.int32), err, 5)
    out["k_reduce_sums"], out["k_reduce_amax"], out["k_reduce_aval"] = s_, i_, v_

    # dithered initial masks (spatial.py:123-148, dither="random")
    for hh, ww, cc, seed in ((64, 64, 3, 0), (96, 80, 1, 7), (128, 128, 3, 2)):
        f = synth(hh, ww, cc, seed)
        n = hh * ww
        init, _ = _schedule(int(0.05 * n), 20, 1.0, None)
        m = sp.analytic_mask(sp.Image(f), init / n, dither="random", sigma=1.0, seed=seed,
                             count=init).indicator
        out[f"initmask_{hh}x{ww}x{cc}_s{seed}"] = m
    t64 = sp.Image(textured64()[None])
    out["initmask_textured64_d007_s5"] = sp.analytic_mask(t64, 0.07, dither="random",
                                                          seed=5).indicator
    out["aamask_textured64_d005"] = sp.analytic_mask(t64, 0.05).indicator

    # densification lockstep trace (64x64 RGB synth, 10 iterations, seed 0)
    f = synth(64, 64, 3, 0)
    trace = []
    orig_acc = sp.spatial.accumulate_errors

    def acc_hook(mesh, error_map, labels):
        ce = orig_acc(mesh, error_map, labels)
        trace.append(dict(labels=labels.labels.copy(), tris=mesh.triangles.copy(),
                          err=np.asarray(error_map).copy(), sums=ce.sums.copy(),
                          amax=ce.argmax_flat.copy()))
        return ce

    sp.spatial.accumulate_errors = acc_hook
    cfg = sp.DensificationConfig(density=0.05, iterations=10, seed=0)
    mask, u, hist = sp.delaunay_densify(sp.Image(f), cfg)
    sp.spatial.accumulate_errors = orig_acc
    for it in (0, 4, 9):
        for k, v in trace[it].items():
            out[f"dd_it{it}_{k}"] = v
    out["dd_final_mask"] = mask.indicator
    sc["dd_history_mse"] = [float(hh[2]) for hh in hist]

    # tonal on the densified mask
    img = sp.Image(f)
    vi = sp.voronoi_richardson_init(img, mask)
    ras = sp.ras_tonal(img, mask, init=vi)
    cg = sp.cgnr_tonal(img, mask)
    sc.update(vi_mse=vi.mse, vi_steps=vi.iterations, ras_mse=ras.mse,
              ras_outer=ras.iterations, cgnr_mse=cg.mse, cgnr_iters=cg.iterations)
    out["tonal_ras_g"] = ras.g.data.astype(np.float32)

    # inpaint (f64 tight) on a 48x40 RGB instance
    f = synth(48, 40, 3, 5)
    m = (np.random.default_rng(9).random((48, 40)) < 0.08).astype(np.uint8)
    u, rep = sp.inpaint(sp.Image(f), sp.Mask(m), sp.MultigridConfig(dtype="float64",
                                                                     tol=1e-10,
                                                                     max_cycles=200))
    out["inpaint_48x40_u"] = u.data
    sc["inpaint_48x40_iters"] = rep.iterations

    # recorded CLI runs of the reference (pkg/test_output.txt:64-71; test_cli.py:87-135)
    sc["recorded"] = {
        "textured64_dd_none": {"density": 0.05, "iterations": 6, "seed": 1, "tonal": "none",
                               "mse": 41.389365, "psnr": 31.9619},
        "textured64_dd_rasvi": {"density": 0.05, "iterations": 6, "seed": 1,
                                "tonal": "ras+vi", "mse": 18.226157, "psnr": 35.5239},
        "textured64_dd_vi": {"density": 0.04, "iterations": 4, "seed": 11,
                             "tonal": "voronoi-init", "mse": 29.5767, "psnr": 33.4213},
    }
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    with open(os.path.join(HERE, "reference_scalars.json"), "w") as fh:
        json.dump(sc, fh, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
