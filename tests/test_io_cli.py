"""Frame ingest/egress formats and the lorbpano CLI on the B200 path
(SURVEY §8(f) rows 3-4): load_pnm / save_pnm (image.hpp:88-204) through the
C-ABI with the reference's error classes, the PPM sink's gray->RGB
triplication on the device (cli.hpp:138-145), the config parser's errors
(config.hpp:84-226) and `stitch` / `extract` / `bench` end to end."""
import os

import numpy as np
import pytest

from paper_1810_03988_b200 import cli, lib
from paper_1810_03988_b200.abi import LorbError


def test_pnm_round_trip_and_comments(tmp_path):
    rng = np.random.default_rng(0)
    g = rng.integers(0, 256, (31, 47), dtype=np.uint8)
    c = rng.integers(0, 256, (9, 5, 3), dtype=np.uint8)
    lib.save_pnm(tmp_path / "g.pgm", g)
    lib.save_pnm(tmp_path / "c.ppm", c)
    assert open(tmp_path / "g.pgm", "rb").read(12) == b"P5\n47 31\n255"
    assert np.array_equal(lib.load_pnm(tmp_path / "g.pgm"), g)
    assert np.array_equal(lib.load_pnm(tmp_path / "c.ppm"), c)
    # '#' comments between header tokens (pnm_read_token, image.hpp:88-103)
    (tmp_path / "k.pgm").write_bytes(b"P5\n# made by hand\n3 # width\n2\n255\n" + bytes(range(6)))
    assert np.array_equal(lib.load_pnm(tmp_path / "k.pgm"), np.arange(6, dtype=np.uint8).reshape(2, 3))


@pytest.mark.parametrize("data,name", [
    (b"P3\n2 2\n255\n0 0 0 0", "UnsupportedFormat"),
    (b"P5\n2 2\n65535\n" + bytes(8), "UnsupportedFormat"),
    (b"P5\n0 2\n255\n", "CorruptData"),
    (b"P5\n4 4\n255\n" + bytes(7), "CorruptData"),
])
def test_pnm_errors(tmp_path, data, name):
    (tmp_path / "x.pgm").write_bytes(data)
    with pytest.raises(LorbError) as e:
        lib.load_pnm(tmp_path / "x.pgm")
    assert e.value.name == name


def test_pnm_missing_and_bad_channels(tmp_path):
    with pytest.raises(LorbError) as e:
        lib.load_pnm(tmp_path / "none.pgm")
    assert e.value.name == "FileNotFound"
    with pytest.raises(LorbError) as e:
        lib.save_pnm(tmp_path / "two.pgm", np.zeros((2, 2, 2), np.uint8))
    assert e.value.name == "UnsupportedFormat"


@pytest.mark.parametrize("text,kind", [
    ("bogus = 1\n", "ValidationError"),
    ("overlap = abc\n", "ParseError"),
    ("[lens]\n", "ParseError"),
    ("overlap = 0\n", "ValidationError"),
    ("[camera]\ncrop = 1,2,3\n", "ValidationError"),
    ("[camera]\nframes = /nonexistent/*.pgm\n", "MissingFrames"),
])
def test_config_errors(tmp_path, text, kind):
    (tmp_path / "c.cfg").write_text(text)

    class _P:  # parse_config only needs default_params()
        def default_params(self):
            from paper_1810_03988_b200 import abi
            import ctypes
            p = abi.Params()
            lib.load().lp_params_default(ctypes.byref(p))
            return p
    with pytest.raises(cli.ConfigError) as e:
        cli.parse_config(str(tmp_path / "c.cfg"), _P())
    assert e.value.kind == kind


def _rig_files(tmp_path, ncams=2, w=640, h=480, frames=2):
    shift = int(np.floor(w * 0.75 + 0.5))
    wide = cli._texture(w + shift * (ncams - 1), h, 42)
    cams = [np.ascontiguousarray(wide[:, c * shift:c * shift + w]) for c in range(ncams)]
    for c in range(ncams):
        for f in range(frames):
            lib.save_pnm(tmp_path / f"cam{c}_{f:03d}.pgm", cams[c])
    cfg = "seed = 42\noverlap = 0.25\nemit_timings = true\n" + "".join(
        f"[camera]\nframes = {tmp_path}/cam{c}_*.pgm\n" for c in range(ncams))
    (tmp_path / "rig.cfg").write_text(cfg)
    return cams


@pytest.mark.gpu
def test_gray_to_rgb(lp):
    g = np.random.default_rng(3).integers(0, 256, (37, 101), dtype=np.uint8)
    assert np.array_equal(lp.gray_to_rgb(g), np.repeat(g[:, :, None], 3, axis=2))


@pytest.mark.gpu
def test_cli_stitch(tmp_path, lp):
    cams = _rig_files(tmp_path)
    assert cli.main(["stitch", "--config", str(tmp_path / "rig.cfg"), "--out", str(tmp_path / "out")]) == 0
    p = lp.default_params()
    p.seed = p.matching.seed = p.prosac.seed = 42
    want = lp.stitch_frame(cams, p, frame_index=0)["panorama"]
    got = lib.load_pnm(tmp_path / "out" / "pano_0.ppm")
    assert np.array_equal(got, np.repeat(want[:, :, None], 3, axis=2))
    rows = open(tmp_path / "out" / "timings.csv").read().splitlines()
    assert rows[0] == "frame_index,stage,duration_ns"
    assert sum(r.startswith("summary,") for r in rows) == 7 and len(rows) == 1 + 2 * 7 + 7


@pytest.mark.gpu
def test_cli_extract_and_bench(tmp_path, lp):
    img = cli._texture(200, 150, 5)
    lib.save_pnm(tmp_path / "img.pgm", img)
    assert cli.main(["extract", str(tmp_path / "img.pgm"), "--seed", "7", "--out", str(tmp_path)]) == 0
    lines = open(tmp_path / "features.csv").read().splitlines()
    p = lp.default_params()
    pairs = lp.brief_pattern(p.extraction.n_d, p.extraction.patch_half, 7)
    kp, _ = lp.extract_features(img, [(15, 15, 185, 135, 0)], p.extraction, pairs)
    assert lines[0] == "x,y,response,region_id,gt_plane,lt_plane" and len(lines) == 1 + len(kp)
    assert cli.main(["bench", "match", "--out", str(tmp_path)]) == 0
    r = open(tmp_path / "bench_match.csv").read().splitlines()
    assert r[0] == "queries,recall,lsh_ms_total,brute_ms_total" and float(r[1].split(",")[1]) >= 0.9
    assert cli.main(["bench", "nope", "--out", str(tmp_path)]) == 2
