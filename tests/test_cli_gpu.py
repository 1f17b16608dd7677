"""The batch frontend (cli.py parity) and the device PNM
encoders (8(f) f2): the reference's TestOptimizeCommand / TestMaskAndTonal /
CSV schema cases (test_cli.py:62-160), and device-encoded file bodies equal
to the host numpy encoders byte for byte."""

import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import paper_2401_06747_b200 as sp
    return sp


def _run(argv):
    from paper_2401_06747_b200 import cli
    return cli.main(argv)


def test_optimize_artifacts_schema_and_exact_count(sp, tmp_path, textured64):
    ipath = str(tmp_path / "t.pgm")
    sp.write_image(ipath, sp.Image(textured64))
    prefix = str(tmp_path / "out")
    rc = _run(["optimize", "--input", ipath, "--output-prefix", prefix, "--density", "0.05",
               "--iterations", "6", "--seed", "1", "--deterministic-output"])
    assert rc == 0
    for suffix in (".mask.pbm", ".values.pgm", ".values16.pgm", ".recon.pgm", ".spatial.csv",
                   ".tonal.csv"):
        assert os.path.exists(prefix + suffix), suffix
    assert sp.read_mask(prefix + ".mask.pbm").count == int(0.05 * 64 * 64)
    lines = open(prefix + ".spatial.csv").read().splitlines()
    assert lines[0] == "iteration,mask_count,mse,psnr,seconds"
    assert len(lines) == 1 + 7 and all(l.endswith(",0.0") for l in lines[1:])
    assert open(prefix + ".tonal.csv").readline().strip() == \
        "iteration,mse,psnr,seconds,inner_solves"


def test_seeded_reruns_are_byte_identical(sp, tmp_path, textured64, capsys):
    ipath = str(tmp_path / "t.pgm")
    sp.write_image(ipath, sp.Image(textured64))
    outs = []
    for k in range(2):
        prefix = str(tmp_path / f"r{k}")
        assert _run(["optimize", "--input", ipath, "--output-prefix", prefix, "--density",
                     "0.04", "--iterations", "4", "--seed", "11", "--tonal", "voronoi-init",
                     "--deterministic-output"]) == 0
        outs.append({s: open(prefix + s, "rb").read()
                     for s in (".mask.pbm", ".values.pgm", ".values16.pgm", ".recon.pgm",
                               ".spatial.csv", ".tonal.csv")})
    assert outs[0] == outs[1]
    printed = capsys.readouterr().out.strip().splitlines()
    assert printed[0] == printed[1] and printed[0].endswith(",0.0")
    assert printed[0].startswith("0.04,dd,voronoi-init,")


def test_mask_then_tonal_commands(sp, tmp_path, textured64, capsys):
    """test_cli.py:120-138 (aa mask -> balance tonal)."""
    ipath = str(tmp_path / "t64.pgm")
    sp.write_image(ipath, sp.Image(textured64))
    mpath = str(tmp_path / "m.pbm")
    assert _run(["mask", "--input", ipath, "--output", mpath, "--density", "0.05",
                 "--spatial", "aa"]) == 0
    assert sp.read_mask(mpath).count == 204
    assert _run(["tonal", "--input", ipath, "--mask", mpath, "--output-values",
                 str(tmp_path / "g.pgm"), "--output-recon", str(tmp_path / "r.pgm"), "--csv",
                 str(tmp_path / "t.csv"), "--tonal", "balance"]) == 0
    assert os.path.exists(tmp_path / "g.pgm.wide")
    assert open(tmp_path / "t.csv").readline().strip() == \
        "iteration,mse,psnr,seconds,inner_solves"
    out = capsys.readouterr().out
    assert "mask_count=204" in out and "mse=40.8392" in out


def test_usage_errors_exit_two(tmp_path):
    assert _run(["eval", str(tmp_path / "missing.pgm"), str(tmp_path / "x.pgm")]) == 2
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("no_such_key = 1\n")
    assert _run(["optimize", "--input", "x.pgm", "--output-prefix", "o", "--config",
                 str(cfg)]) == 2


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("c,h,w", [(1, 37, 29), (3, 64, 70), (3, 5, 9)])
def test_device_pnm_bodies_equal_host_encoders(sp, tmp_path, dtype, c, h, w):
    import torch
    rng = np.random.default_rng(c * h + w)
    v = rng.uniform(-300, 600, (c, h, w)).astype(dtype)
    v.ravel()[:8] = [-0.5, 0.5, 1.5, 2.5, 254.5, 255.5, -256.0, 767.99][:8]
    m = (rng.random((h, w)) < 0.3).astype(np.uint8)
    dev_v = sp.Image(torch.from_numpy(v).cuda())
    dev_m = sp.Mask(torch.from_numpy(m).cuda())
    assert dev_v.on_device and dev_m.on_device
    for name, fn in (("img", lambda p, a, b: sp.write_image(p, a)),
                     ("tonal8", lambda p, a, b: sp.write_tonal(p, a, b)),
                     ("tonal16", lambda p, a, b: sp.write_tonal(p, a, b, wide=True)),
                     ("mask", lambda p, a, b: sp.write_mask(p, b))):
        pd, ph = str(tmp_path / f"{name}_d"), str(tmp_path / f"{name}_h")
        fn(pd, dev_v, dev_m)
        fn(ph, sp.Image(v), sp.Mask(m))
        assert open(pd, "rb").read() == open(ph, "rb").read(), name
    # and the round trip
    assert np.array_equal(sp.read_mask(str(tmp_path / "mask_d")).indicator, m)
    back = sp.read_tonal(str(tmp_path / "tonal16_d"), wide=True).data
    enc = np.where(m[None] > 0, v, 0).astype(np.float64)
    inside = (enc > -256) & (enc < 767.98)
    # half a 1/64 step, plus the float32 rounding of (v + 256) * 64
    assert np.all(np.abs(back - enc)[inside] <= 1 / 128 + 1e-4)


def test_synth_roundtrip_via_cli_eval(sp, tmp_path, capsys):
    f = O.synth(40, 48, 3, 2)
    a, b = str(tmp_path / "a.ppm"), str(tmp_path / "b.ppm")
    sp.write_image(a, sp.Image(f))
    sp.write_image(b, sp.Image(f))
    assert _run(["eval", a, b]) == 0
    assert "psnr=exact" in capsys.readouterr().out
