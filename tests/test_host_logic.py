"""Host-side logic of the product package (no GPU): configs and their
validation, budget schedule, block decomposition, JFA step schedule, PCG64
seeding, Gaussian weights, PNM codecs.  Mirrors the reference's unit tests
(test_spatial.py:53-73, test_solver.py:49-80, test_geometry.py, test_pnm.py)."""

import math

import numpy as np
import pytest

import paper_2401_06747_b200 as sp
from paper_2401_06747_b200 import geometry, spatial
from oracle import oracle as O


class TestSchedule:
    def test_constant_growth_splits_evenly(self):
        init, counts = spatial._schedule(204, 10, 1.0, None)
        assert init + sum(counts) == 204 and init == 19 and counts[:-1] == [18] * 9

    def test_growth_factor_increases_counts(self):
        init, counts = spatial._schedule(500, 8, 1.2, None)
        assert init + sum(counts) == 500
        assert all(b >= a for a, b in zip(counts[:-2], counts[1:-1]))

    def test_explicit_initial_fraction(self):
        assert spatial._schedule(100, 5, 1.0, 0.5)[0] == 50

    def test_initial_share_consumes_everything(self):
        init, counts = spatial._schedule(50, 5, 1.0, 1.0)
        assert init == 50 and sum(counts) == 0

    @pytest.mark.parametrize("total,it,g", [(414720, 20, 1.0), (52428, 20, 1.0), (3276, 7, 1.3)])
    def test_matches_oracle(self, total, it, g):
        assert spatial._schedule(total, it, g, None) == O.schedule(total, it, g, None)

    def test_4k_budget(self):
        # 414,720 / 19,749 / 19,748 (last 19,759)
        init, counts = spatial._schedule(int(0.05 * 3840 * 2160), 20, 1.0, None)
        assert init == 19749 and counts[0] == 19748 and counts[-1] == 19759


class TestDecomposition:
    @pytest.mark.parametrize("block,overlap", [(32, 6), (64, 6)])
    @pytest.mark.parametrize("shape", [(32, 32), (50, 70), (128, 96), (33, 65), (20, 20),
                                       (1, 40)])
    def test_partition_of_unity_is_exact(self, shape, block, overlap):
        d = sp.build_decomposition(shape[0], shape[1], block, overlap)
        assert np.all(d.weight_sums() == 1.0)

    def test_block_count_follows_stride(self):
        d = sp.build_decomposition(2160, 3840, 32, 6)
        assert d.ys.size == 83 and d.xs.size == 148

    def test_weights_match_oracle(self):
        d = sp.build_decomposition(37, 29, 16, 4)
        assert np.array_equal(d.weights, O.build_decomposition(37, 29, 16, 4)["weights"])

    def test_invalid_configs_rejected(self):
        with pytest.raises(ValueError):
            sp.OrasConfig(block=6, overlap=6)
        with pytest.raises(ValueError):
            sp.OrasConfig(overlap=0)
        with pytest.raises(ValueError):
            sp.OrasConfig(rho=1.5)
        with pytest.raises(ValueError):
            sp.MultigridConfig(pre=0, post=0)
        with pytest.raises(ValueError):
            sp.MultigridConfig(dtype="float16")
        with pytest.raises(ValueError):
            sp.DensificationConfig(density=0.0)
        with pytest.raises(ValueError):
            sp.RasTonalConfig(block=6, overlap=6)
        with pytest.raises(ValueError):
            sp.InitConfig(tau=0)

    def test_robin_gamma_default_is_dirichlet(self):
        assert sp.OrasConfig().robin_gamma() == 0.0


class TestSchedulesAndSeeds:
    @pytest.mark.parametrize("dim,hint", [(64, None), (3840, None), (4320, 12.3), (8, 1.0),
                                          (1, None), (512, 600.0)])
    def test_jfa_steps_match_oracle(self, dim, hint):
        assert np.array_equal(geometry.steps_for(dim, hint), O.steps_for(dim, hint))

    def test_jfa_schedule_shape(self):
        # extra unit step first, then halving (geometry.py:84-89)
        assert geometry.steps_for(512, None).tolist() == [1, 256, 128, 64, 32, 16, 8, 4, 2, 1]

    def test_pcg_state_roundtrip(self):
        st = spatial._pcg_state(7)
        ref = np.random.default_rng(7).bit_generator.state["state"]
        assert (int(st[1]) << 64 | int(st[0])) == ref["state"]
        assert (int(st[3]) << 64 | int(st[2])) == ref["inc"]

    def test_gaussian_weights_equal_scipy(self):
        from scipy.ndimage import _filters
        w, r = spatial._gaussian_weights(1.0)
        ref = _filters._gaussian_kernel1d(1.0, 0, 4)[::-1]
        assert r == 4 and np.array_equal(w, ref)

    def test_pcg64_host_advance_matches_numpy(self):
        """Host restatement of the device jump-ahead (csrc/dither.cu)."""
        M = 0x2360ED051FC65DA44385DF649FCCF645
        st = np.random.default_rng(3).bit_generator.state["state"]
        s, inc = st["state"], st["inc"]
        out = []
        for _ in range(5):
            s = (s * M + inc) % (1 << 128)
            rot = s >> 122
            x = ((s >> 64) ^ s) & ((1 << 64) - 1)
            v = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
            out.append((v >> 11) * (1.0 / 9007199254740992.0))
        assert out == np.random.default_rng(3).random(5).tolist()


class TestContainers:
    def test_image_promotes_and_validates(self):
        img = sp.Image(np.ones((4, 5), dtype=np.uint8))
        assert img.shape == (1, 4, 5) and img.data.dtype == np.float64
        with pytest.raises(ValueError):
            sp.Image(np.full((2, 2), np.nan))
        with pytest.raises(ValueError):
            sp.Image(np.zeros((1, 1, 2, 2)))

    def test_mask_binarizes(self):
        m = sp.Mask(np.array([[0, 2], [5, 0]]))
        assert m.indicator.tolist() == [[0, 1], [1, 0]] and m.count == 2

    def test_quality_report(self):
        q = sp.QualityReport(mse=0.0)
        assert q.exact and q.psnr == math.inf
        assert abs(sp.QualityReport(mse=65.025).psnr - 30.0) < 1e-9


class TestPnm:
    def test_roundtrips(self, tmp_path):
        rng = np.random.default_rng(0)
        img = sp.Image(rng.integers(0, 256, (3, 7, 5)).astype(np.float64))
        sp.write_image(tmp_path / "a.ppm", img)
        assert np.array_equal(sp.read_image(tmp_path / "a.ppm").data, img.data)
        m = sp.Mask(rng.random((9, 13)) < 0.3)
        sp.write_mask(tmp_path / "m.pbm", m)
        assert np.array_equal(sp.read_mask(tmp_path / "m.pbm").indicator, m.indicator)
        vals = sp.Image(rng.uniform(-100, 600, (1, 9, 13)))
        sp.write_tonal(tmp_path / "t.pgm", vals, m, wide=True)
        back = sp.read_tonal(tmp_path / "t.pgm", wide=True).data
        expect = np.where(m.indicator[None].astype(bool), vals.data, 0.0)
        assert np.abs(back - expect).max() <= 1 / 128


def test_pipeline_config_mirrors_reference_defaults():
    cfg = sp.PipelineConfig()
    assert (cfg.density, cfg.spatial, cfg.tonal, cfg.iterations) == (0.05, "dd", "ras+vi", 20)
    assert cfg.solver().cfg.tol == 1e-4 and cfg.ras().local_product_tol == 1e-2
    with pytest.raises(ValueError):
        sp.PipelineConfig(spatial="bogus").validate()
