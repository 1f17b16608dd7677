"""Densification geometry on the GPU: bit-exact against the reference
fixtures and the oracle.  The north_star contract: Voronoi labels, dithered
masks and triangulation indices bit-exact for the same error map and seed
(checked in lockstep, feeding the reference's own per-iteration
mask + error map)."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_vectors.npz"))


@pytest.fixture(scope="module")
def sp():
    import paper_2401_06747_b200 as sp
    return sp


@pytest.mark.parametrize("hh,ww,cc,seed", [(64, 64, 3, 0), (96, 80, 1, 7), (128, 128, 3, 2)])
def test_dithered_initial_mask_matches_reference(sp, hh, ww, cc, seed):
    from paper_2401_06747_b200 import spatial
    f = O.synth(hh, ww, cc, seed)
    n = hh * ww
    init, _ = spatial._schedule(int(0.05 * n), 20, 1.0, None)
    m = sp.analytic_mask(sp.Image(f), init / n, dither="random", sigma=1.0, seed=seed,
                         count=init)
    assert np.array_equal(m.indicator, G[f"initmask_{hh}x{ww}x{cc}_s{seed}"])


def test_dithered_masks_textured_and_fs(sp, textured64):
    img = sp.Image(textured64)
    assert np.array_equal(sp.analytic_mask(img, 0.07, dither="random", seed=5).indicator,
                          G["initmask_textured64_d007_s5"])
    assert np.array_equal(sp.analytic_mask(img, 0.05).indicator, G["aamask_textured64_d005"])


@pytest.mark.parametrize("shape,seed", [((1, 512, 384), 3), ((3, 300, 301), 11)])
def test_dithered_mask_vs_oracle_larger(sp, shape, seed):
    f = O.synth(shape[1], shape[2], shape[0], seed)
    n = shape[1] * shape[2]
    init = max(1, int(0.05 * n) // 21)
    got = sp.analytic_mask(sp.Image(f), init / n, dither="random", seed=seed,
                           count=init).indicator
    assert np.array_equal(got, O.analytic_mask(f, init / n, dither="random", seed=seed,
                                               count=init))


def test_constant_image_falls_back_to_uniform(sp):
    m = sp.analytic_mask(sp.Image(np.full((1, 16, 16), 9.0)), 0.1, seed=3)
    assert m.count == 25
    assert np.array_equal(m.indicator, O.uniform_random_mask(16, 16, 25, 3))


def test_pcg64_stream_and_pairwise_sum(sp):
    import ctypes
    from paper_2401_06747_b200 import _lib, spatial
    st = spatial._pcg_state(42)
    out = torch.empty(5000, dtype=torch.float64, device="cuda")
    _lib.call("sp_pcg64_doubles", _lib.ptr(st), 1234, 5000, _lib.ptr(out), _lib.stream())
    ref = np.random.default_rng(42).random(6234)[1234:]
    assert np.array_equal(out.cpu().numpy(), ref)
    for n in (7, 128, 129, 1000, 4321, 2160 * 3840):
        a = np.abs(np.random.default_rng(n).standard_normal(n)) * 1e3
        tot = ctypes.c_double()
        _lib.call("sp_pairwise_sum", _lib.ptr(torch.from_numpy(a).cuda()), n,
                  ctypes.byref(tot), _lib.stream())
        assert tot.value == float(a.sum()), n


_TRACE = {}


def _oracle_trace():
    """Per-iteration (mask, error map, labels, triangles, picks) of the
    oracle densification -- bit-exact with the reference (the CPU test
    test_oracle_golden.py pins iterations 0/4/9 against the fixtures)."""
    if not _TRACE:
        trace = []
        O.delaunay_densify(O.synth(64, 64, 3, 0), 0.05, 10, seed=0, trace=trace)
        _TRACE.update(enumerate(trace))
    return _TRACE


def test_lockstep_picks_match_oracle(sp):
    """Every densification iteration: same error map in -> same picks out."""
    from paper_2401_06747_b200.geometry import workspace
    t = _oracle_trace()
    ws = workspace(64, 64)
    hint = None
    for i in sorted(t):
        mask_t = torch.from_numpy(t[i]["mask"].astype(np.uint8)).cuda()
        ws.voronoi(mask_t, hint)
        hint = ws.max_radius
        assert np.array_equal(ws.labels_tensor().cpu().numpy(), t[i]["labels"])
        nb = ws.delaunay()
        assert np.array_equal(ws.triangles_tensor().cpu().numpy(), t[i]["tris"])
        ws.accumulate(torch.from_numpy(t[i]["err"]).cuda())
        sums, amax, _ = ws.buckets(nb)
        assert np.array_equal(sums.cpu().numpy(), t[i]["sums"])
        assert np.array_equal(amax.cpu().numpy(), t[i]["amax"])
        if i in (0, 4, 9):  # the reference's own arrays
            assert np.array_equal(ws.triangles_tensor().cpu().numpy(), G[f"dd_it{i}_tris"])
            assert np.array_equal(sums.cpu().numpy(), G[f"dd_it{i}_sums"])
        picked = ws.select(mask_t, nb, t[i]["want"])
        assert picked == len(t[i]["picked"])
        expect = t[i]["mask"].copy().ravel()
        expect[t[i]["picked"]] = 1
        assert np.array_equal(mask_t.cpu().numpy().ravel(), expect)


def test_jfa_against_oracle_with_hints(sp):
    rng = np.random.default_rng(11)
    for (h, w, d) in ((300, 257, 0.01), (128, 128, 0.002), (1, 40, 0.1), (64, 64, 0.3)):
        m = (rng.random((h, w)) < d).astype(np.uint8)
        m.ravel()[rng.integers(0, h * w)] = 1
        for hint in (None, 3.0, 40.0):
            lab = sp.jump_flood_voronoi(sp.Mask(m), hint)
            lo, seeds, rad = O.jump_flood_voronoi(m, hint)
            assert np.array_equal(lab.labels, lo) and lab.max_radius == rad
            if (lo < 0).any():
                # a too-small hint leaves pixels unlabelled (-1); the densify
                # loop never triangulates such a map (its hint is the
                # previous, larger radius), so only the labels are pinned
                continue
            mesh = sp.delaunay_from_voronoi(lab)
            to, eo = O.delaunay_from_voronoi(lo, seeds.shape[0])
            assert np.array_equal(mesh.triangles, to)
            assert np.array_equal(mesh.edges, eo)


@pytest.mark.parametrize("short4", [0, 1])
def test_jfa_short_steps_on_quads_match_oracle(sp, short4):
    """Passes of step 1 and 2 on pixel quads (k_jfa_pass_key4s: aligned
    16-byte candidate loads, out-of-image candidates as the phantom key) and
    per pixel (k_jfa_pass_key): labels equal to the oracle's bit for bit, on
    widths that are multiples of 4 (the quad kernel's domain) incl. the
    image edges."""
    from paper_2401_06747_b200 import _lib
    lib = _lib.load()
    prev = lib.sp_jfa_short4(-1)
    rng = np.random.default_rng(12)
    try:
        lib.sp_jfa_short4(short4)
        for (h, w, d) in ((96, 160, 0.02), (37, 52, 0.1), (8, 4, 0.3), (200, 256, 0.005)):
            m = (rng.random((h, w)) < d).astype(np.uint8)
            m.ravel()[rng.integers(0, h * w)] = 1
            for hint in (None, 1.0, 2.0, 6.0):
                lab = sp.jump_flood_voronoi(sp.Mask(m), hint)
                lo, _, rad = O.jump_flood_voronoi(m, hint)
                assert np.array_equal(lab.labels, lo) and lab.max_radius == rad
    finally:
        lib.sp_jfa_short4(prev)


def test_reference_geometry_kats(sp):
    """test_geometry.py:24-103 known answers."""
    def mask_from(h, w, pts):
        m = np.zeros((h, w), np.uint8)
        for y, x in pts:
            m[y, x] = 1
        return sp.Mask(m)
    lab = sp.jump_flood_voronoi(mask_from(1, 8, [(0, 0), (0, 7)]))
    assert lab.labels[0].tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    mesh = sp.delaunay_from_voronoi(sp.jump_flood_voronoi(
        mask_from(16, 16, [(2, 2), (3, 13), (12, 6)])))
    assert mesh.triangles.tolist() == [[0, 1, 2]] and not mesh.degenerate
    mesh = sp.delaunay_from_voronoi(sp.jump_flood_voronoi(
        mask_from(8, 8, [(1, 1), (1, 6), (6, 1), (6, 6)])))
    assert mesh.triangles.tolist() == [[0, 1, 3], [0, 2, 3]]
    mesh = sp.delaunay_from_voronoi(sp.jump_flood_voronoi(mask_from(8, 8, [(1, 1), (6, 6)])))
    assert mesh.degenerate and mesh.edges.tolist() == [[0, 1]]
    with pytest.raises(ValueError):
        sp.jump_flood_voronoi(sp.Mask(np.zeros((4, 4))))


def test_accumulate_errors_partition_and_kat(sp):
    """test_geometry.py:169-184: sums partition the error; unit-error argmax."""
    rng = np.random.default_rng(2)
    m = (rng.random((48, 48)) < 0.05).astype(np.uint8)
    lab = sp.jump_flood_voronoi(sp.Mask(m))
    mesh = sp.delaunay_from_voronoi(lab)
    err = rng.uniform(0, 1, (48, 48))
    ce = sp.accumulate_errors(mesh, err, lab)
    lo, seeds, _ = O.jump_flood_voronoi(m)
    so, ao, vo, _ = O.accumulate_errors(mesh.triangles, err, lo, seeds)
    assert np.array_equal(ce.sums, so) and np.array_equal(ce.argmax_flat, ao)
    assert abs(ce.total - err.sum()) <= 1e-9 * err.sum()
    s2, a2, _ = sp.voronoi_cell_errors(lab, err)
    s3, a3, _ = O.voronoi_cell_errors(lo, seeds.shape[0], err)
    assert np.array_equal(s2, s3) and np.array_equal(a2, a3)


def test_voronoi_weights_and_cell_average(sp):
    rng = np.random.default_rng(4)
    m = (rng.random((40, 56)) < 0.06).astype(np.uint8)
    lab = sp.jump_flood_voronoi(sp.Mask(m))
    lo, seeds, _ = O.jump_flood_voronoi(m)
    for scheme in ("inverse-log", "constant"):
        w = sp.voronoi_weights(lab, scheme)
        wo = O.voronoi_weights(lo, seeds, scheme)
        assert np.allclose(w, wo, rtol=1e-15, atol=0)
    plane = rng.standard_normal((40, 56))
    a = sp.geometry.cell_weighted_average(lab, wo, plane)
    assert np.array_equal(a, O.cell_weighted_average(lo, seeds.shape[0], wo, plane))


def test_densify_64_matches_reference_end_to_end(sp):
    """At 64x64 RGB the GPU densification reproduces the reference mask."""
    f = O.synth(64, 64, 3, 0)
    mask, u, hist = sp.delaunay_densify(sp.Image(f), sp.DensificationConfig(
        density=0.05, iterations=10, seed=0))
    assert np.array_equal(mask.indicator, G["dd_final_mask"])
    S = json.load(open(os.path.join(HERE, "golden", "reference_scalars.json")))
    assert np.allclose([h[2] for h in hist], S["dd_history_mse"], rtol=1e-4)


@pytest.mark.parametrize("h,w,d,seed", [(64, 64, 0.05, 0), (300, 257, 0.01, 1),
                                        (97, 131, 0.002, 2), (33, 500, 0.2, 3),
                                        (512, 384, 0.05, 4), (70, 70, 0.0005, 5)])
def test_tiled_accumulate_bit_exact(sp, h, w, d, seed):
    """Tile-binned rasteriser + bbox-order reduction (default) vs the global
    atomicMin rasteriser + pixel radix sort and vs the oracle (numba_impl.py:
    442-498): sums, argmax and max values identical, including sparse masks
    whose hull leaves fallback pixels and tiles crossed by large triangles."""
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.geometry import workspace
    rng = np.random.default_rng(seed)
    m = (rng.random((h, w)) < d).astype(np.uint8)
    m.ravel()[rng.choice(h * w, 3, replace=False)] = 1
    err = rng.random((h, w)) * 100.0
    err[rng.random((h, w)) < 0.3] = 0.0          # ties for the argmax order
    lib = _lib.load()
    ws = workspace(h, w)
    got = {}
    try:
        for mode in (0, 1):
            lib.sp_geo_accumulate_mode(mode)
            ws.voronoi(torch.from_numpy(m).cuda())
            nb = ws.delaunay()
            ws.accumulate(torch.from_numpy(err).cuda())
            got[mode] = [x.cpu().numpy() for x in ws.buckets(nb)]
    finally:
        lib.sp_geo_accumulate_mode(1)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b)
    lab, seeds, _ = O.jump_flood_voronoi(m)
    tris, _ = O.delaunay_from_voronoi(lab, seeds.shape[0])
    s, ai, av, _ = O.accumulate_errors(tris, err, lab, seeds)
    assert np.array_equal(got[1][0], s)
    assert np.array_equal(got[1][1], ai)
    assert np.array_equal(got[1][2], av)


class _ThreadGather:
    """all-gather between the threads of one process (one per simulated
    rank), for the StripGeometry partition test"""

    def __init__(self, world):
        import threading
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def for_rank(self, rank):
        outer = self

        class _G:
            def allgather_var(self, t):
                outer.slots[rank] = t.reshape(-1).clone()
                outer.bar.wait()
                got = list(outer.slots)
                outer.bar.wait()
                return got
        return _G()


@pytest.mark.parametrize("shape,dens,P", [((128, 160), 0.05, 2), ((128, 160), 0.004, 3),
                                          ((301, 256), 0.02, 4), ((97, 64), 0.1, 2),
                                          ((2160, 3840), 0.05, 2), ((2160, 3840), 0.0024, 3)])
def test_strip_geometry_bit_identical(shape, dens, P):
    """The row-strip partition of the Delaunay step and the accumulate
    (geometry.StripGeometry: per-strip corner keys merged, per-strip
    rasterisation with the assignment rows gathered, per-rank triangle ranges
    reduced over the full map) gives every rank the unpartitioned triangles
    and buckets bit for bit -- incl. hull-exterior (fallback) pixels of
    sparse masks and uneven strips."""
    import threading
    import torch
    from paper_2401_06747_b200.geometry import GeoWorkspace, StripGeometry
    H, W = shape
    rng = np.random.default_rng(11)
    mask = torch.from_numpy((rng.random((H, W)) < dens).astype(np.uint8)).cuda()
    err = torch.from_numpy(rng.random((H, W)) * 30.0).cuda()
    ref = GeoWorkspace(H, W)
    ref.voronoi(mask)
    T = ref.delaunay()
    ref.accumulate(err)
    tris_ref = ref.triangles_tensor().cpu().numpy()
    b_ref = [x.cpu().numpy() for x in ref.buckets(T)]
    rows = [(H * p // P, H * (p + 1) // P) for p in range(P)]
    comm = _ThreadGather(P)
    wss = [GeoWorkspace(H, W) for _ in range(P)]
    for ws in wss:
        ws.voronoi(mask)
    errs = []

    def run(p):
        try:
            sg = StripGeometry(wss[p], rows, p, comm.for_rank(p))
            assert sg.delaunay() == T
            sg.accumulate(err)
        except Exception as e:  # surfaced below
            errs.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=run, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    for ws in wss:
        assert np.array_equal(ws.triangles_tensor().cpu().numpy(), tris_ref)
        for a, b in zip(ws.buckets(T), b_ref):
            assert np.array_equal(a.cpu().numpy(), b)


@pytest.mark.parametrize("shape,dens", [((128, 160), 0.05), ((97, 64), 0.3)])
def test_delaunay_wide_keys_match_packed(shape, dens):
    """>= 2^21 stored pixels overflow the packed 3 x 21-bit triangle keys;
    sp_geo_delaunay then sorts (a, b << 32 | c) pairs by two stable radix
    passes.  Forced on small masks (sp_geo_wide_threshold), the wide path
    gives the packed path's triangles (np.unique order) and buckets."""
    import torch
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.geometry import GeoWorkspace
    lib = _lib.load()
    H, W = shape
    rng = np.random.default_rng(5)
    mask = torch.from_numpy((rng.random((H, W)) < dens).astype(np.uint8)).cuda()
    err = torch.from_numpy(rng.random((H, W))).cuda()
    out = []
    prev = lib.sp_geo_wide_threshold(0)
    try:
        for thr in (prev, 3):
            lib.sp_geo_wide_threshold(thr)
            ws = GeoWorkspace(H, W)
            ws.voronoi(mask)
            T = ws.delaunay()
            ws.accumulate(err)
            out.append((ws.triangles_tensor().cpu().numpy(),
                        [x.cpu().numpy() for x in ws.buckets(T)]))
    finally:
        lib.sp_geo_wide_threshold(prev)
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a, b)


def test_delaunay_above_2p21_seeds():
    """A mask with more than 2^21 stored pixels (the reference accepts any
    density): the triangulation completes, sorted unique triples of seed
    indices, each triangle's corner pixels really adjacent in the labels."""
    import torch
    from paper_2401_06747_b200.geometry import GeoWorkspace
    H, W = 1536, 1500
    rng = np.random.default_rng(9)
    mask = torch.from_numpy((rng.random((H, W)) < 0.95).astype(np.uint8)).cuda()
    ws = GeoWorkspace(H, W)
    m, _ = ws.voronoi(mask)
    assert m >= 2 ** 21
    T = ws.delaunay()
    tris = ws.triangles_tensor().cpu().numpy().astype(np.int64)
    assert T == tris.shape[0] > 0
    assert (tris[:, 0] < tris[:, 1]).all() and (tris[:, 1] < tris[:, 2]).all()
    assert tris.max() < m
    key = (tris[:, 0] * m + tris[:, 1]) * m + tris[:, 2]
    assert (np.diff(key) > 0).all()          # sorted, unique
