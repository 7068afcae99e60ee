"""GPU parity: the CUDA path (through the C-ABI) against the C restatement
oracle on identical seeded inputs. Integer/byte/index outputs and the FP32
rasters must be bit-identical; homographies are compared bit-exact too (the
device DLT replays the oracle's canonical SVD) with the reference's own
tolerance (frobenius_rel < 1e-4, test_homography.cpp:12-19) as the floor."""
import os

import numpy as np
import pytest

from tests.conftest import chain_cameras, rand_image
from tests.golden.make_golden import prosac_data

pytestmark = pytest.mark.gpu


def frob_rel(a, b):
    a = np.asarray(a, float) / a[2, 2]
    b = np.asarray(b, float) / b[2, 2]
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---------------------------------------------------------------- L-ORB
@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("arc", [9, 12, 16])
def test_fast_corners(lp, orc, seed, arc):
    img = rand_image(97, 83, seed)
    for region, t in (((0, 0, 97, 83, 0), 20), ((10, 7, 60, 70, 1), 5 + seed)):
        a = lp.fast_corners(img, region, t, arc)
        b = orc.fast_corners(img, region, t, arc)
        assert np.array_equal(a, b)


def test_fast_corners_texture_and_cap(lp, orc):
    tex = orc.texture(400, 300, 3)
    a = lp.fast_corners(tex, (15, 15, 385, 285, 0))
    b = orc.fast_corners(tex, (15, 15, 385, 285, 0))
    assert len(a) > 1000 and np.array_equal(a, b)


@pytest.mark.parametrize("sigma", [1.0, 0.7, 1.6])
def test_harris(lp, orc, sigma):
    img = orc.texture(120, 90, 9)
    r = int(np.ceil(3 * sigma)) + 1
    ys, xs = np.mgrid[r:90 - r:3, r:120 - r:2]
    xy = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.int32)
    a = lp.harris_response(img, xy, 0.04, sigma)
    b = orc.harris_response(img, xy, 0.04, sigma)
    assert a.tobytes() == b.tobytes()


def test_nms_topn(lp, orc):
    img = orc.texture(200, 150, 4)
    xy = orc.fast_corners(img, (10, 10, 190, 140, 0))
    resp = orc.harris_response(img, xy)
    kp = np.zeros((len(xy), 4), np.int32)
    kp[:, :2] = xy
    kp[:, 2] = resp.view(np.int32)
    kp[:, 3] = 2
    for radius in (1, 2):
        assert np.array_equal(lp.nms(kp, radius), orc.nms(kp, radius))
    # ties: quantised responses force (y,x) tie-breaks
    kq = kp.copy()
    kq[:, 2] = np.round(resp / 1000.0).astype(np.float32).view(np.int32)
    assert np.array_equal(lp.nms(kq, 1), orc.nms(kq, 1))
    for n in (1, 37, 5000):
        assert np.array_equal(lp.select_top_n(kq, n), orc.select_top_n(kq, n))


def test_select_top_n_and_nms_large(lp, orc):
    """The repo's own compaction and radix sort (csrc/prims.cuh) behind
    lp_nms / lp_select_top_n over many tiles: 300K candidates with heavily
    tied responses and negative coordinates, host and device inputs."""
    import torch
    rng = np.random.default_rng(5)
    n = 300_000
    kp = np.zeros((n, 4), np.int32)
    kp[:, 0] = rng.integers(-50, 1500, n)
    kp[:, 1] = rng.integers(-20, 900, n)
    kp[:, 2] = rng.integers(0, 64, n).astype(np.float32).view(np.int32)
    kp[:, 3] = rng.integers(0, 6, n)
    # unique positions (the reference's grid keeps one candidate per cell)
    _, first = np.unique(kp[:, 0].astype(np.int64) * 4096 + kp[:, 1], return_index=True)
    kp = kp[np.sort(first)]
    for top_n in (1, 777, 50_000, len(kp)):
        assert np.array_equal(lp.select_top_n(kp, top_n), orc.select_top_n(kp, top_n)), top_n
    want = orc.nms(kp, 1)
    assert np.array_equal(lp.nms(kp, 1), want)
    import ctypes as C
    dev = torch.from_numpy(kp).cuda()
    out = np.zeros_like(kp)
    cnt = C.c_int()
    lp._call("nms", C.c_void_p(dev.data_ptr()), len(kp), 1, out.ctypes.data_as(C.c_void_p), C.byref(cnt))
    assert np.array_equal(out[:cnt.value], want)


@pytest.mark.parametrize("sigma,ch", [(1.0, 1), (2.0, 1), (1.5, 3)])
def test_gaussian_blur(lp, orc, sigma, ch):
    rng = np.random.default_rng(1)
    shape = (61, 77) if ch == 1 else (61, 77, ch)
    img = rng.uniform(0, 255, size=shape).astype(np.float32)
    assert lp.gaussian_blur(img, sigma).tobytes() == orc.gaussian_blur(img, sigma).tobytes()


def test_brief_descriptors(lp, orc):
    img = orc.texture(160, 120, 2).astype(np.float32)
    sm = orc.gaussian_blur(img, 2.0)
    pat = orc.brief_pattern(256, 15, 42)
    kp = np.array([[x, y, 0, 0] for x in range(15, 145, 13) for y in range(15, 105, 11)], np.int32)
    assert np.array_equal(lp.brief_descriptors(sm, kp, pat), orc.brief_descriptors(sm, kp, pat))
    pat512 = orc.brief_pattern(512, 15, 7)
    assert np.array_equal(lp.brief_descriptors(sm, kp, pat512), orc.brief_descriptors(sm, kp, pat512))


@pytest.mark.parametrize("w,h", [(640, 480), (1920, 1080)])
def test_extract_features(lp, orc, params, w, h):
    l, r, _ = orc.planted_pair(w, h, 0.25, 42)
    regs = orc.partition_regions([(w, h), (w, h)], 0.25, 15)
    pat = orc.brief_pattern(256, 15, 42)
    for img, rg in ((l, regs[:1]), (r, regs[1:]), (l, regs)):
        ka, da = lp.extract_features(img, rg, params.extraction, pat)
        kb, db = orc.extract_features(img, rg, params.extraction, pat)
        assert len(ka) == len(kb) > 0
        assert np.array_equal(ka, kb)
        assert np.array_equal(da, db)


def test_extract_features_full_frame_region(lp, orc, params):
    """A full-image region (cmd_extract, cli.hpp:172-207) with more survivors
    than top_n in many radix buckets."""
    img = orc.texture(800, 600, 11)
    cfg = params.extraction
    pat = orc.brief_pattern(cfg.n_d, cfg.patch_half, 42)
    reg = [(15, 15, 785, 585, 0)]
    ka, da = lp.extract_features(img, reg, cfg, pat)
    kb, db = orc.extract_features(img, reg, cfg, pat)
    assert np.array_equal(ka, kb) and np.array_equal(da, db)


@pytest.mark.parametrize("top_n", [4, 37, 2048, 3000])
def test_extract_top_n_paths(lp, orc, params, top_n):
    """Histogram + rank top-N (top_n <= 2048) and the radix/bitonic path (> 2048)."""
    from oracle.oracle import Oracle  # noqa: F401
    img = orc.texture(700, 500, 13)
    cfg = orc.default_params().extraction
    cfg.top_n = top_n
    pat = orc.brief_pattern(cfg.n_d, cfg.patch_half, 42)
    reg = [(15, 15, 685, 485, 0), (100, 40, 300, 200, 0)]
    ka, da = lp.extract_features(img, reg, cfg, pat)
    kb, db = orc.extract_features(img, reg, cfg, pat)
    assert np.array_equal(ka, kb) and np.array_equal(da, db)


def test_extract_widened_parameter_domain(lp, orc):
    """ExtractionConfig::validate (lorb.hpp:82-89) accepts any sigma > 0 and
    top_n >= 4. The device covers harris_sigma <= 4 (generic detect tile),
    brief_blur_sigma <= 8 and any top_n (> 8192: the global radix-sort top-N
    path); beyond the two sigma bounds it raises BadParams (tested below)."""
    img = orc.texture(1920, 1080, 21)
    reg = [(20, 20, 1900, 1060, 0)]
    for hs, bs, top_n in ((3.5, 2.0, 500), (4.0, 2.0, 500), (1.0, 6.0, 300), (1.0, 2.0, 9000), (2.6, 5.5, 12000)):
        cfg = orc.default_params().extraction
        cfg.harris_sigma, cfg.brief_blur_sigma, cfg.top_n = hs, bs, top_n
        pat = orc.brief_pattern(cfg.n_d, cfg.patch_half, 42)
        ka, da = lp.extract_features(img, reg, cfg, pat)
        kb, db = orc.extract_features(img, reg, cfg, pat)
        assert len(ka) == len(kb) > 0, (hs, bs, top_n)
        assert np.array_equal(ka, kb), (hs, bs, top_n)
        assert np.array_equal(da, db), (hs, bs, top_n)
    from paper_1810_03988_b200 import abi
    for hs, bs in ((4.2, 2.0), (1.0, 8.5)):
        cfg = orc.default_params().extraction
        cfg.harris_sigma, cfg.brief_blur_sigma = hs, bs
        pat = orc.brief_pattern(cfg.n_d, cfg.patch_half, 42)
        with pytest.raises(abi.LorbError) as e:
            lp.extract_features(img, reg, cfg, pat)
        assert e.value.name == "BadParams", e.value.name


# ---------------------------------------------------------------- matching
def _descs(orc, params, w=640, h=480):
    l, r, _ = orc.planted_pair(w, h, 0.25, 42)
    regs = orc.partition_regions([(w, h), (w, h)], 0.25, 15)
    pat = orc.brief_pattern(256, 15, 42)
    _, dl = orc.extract_features(l, regs[:1], params.extraction, pat)
    _, dr = orc.extract_features(r, regs[1:], params.extraction, pat)
    return dl, dr


def test_match_features(lp, orc, params):
    dl, dr = _descs(orc, params)
    mc = params.matching
    a = lp.match_features(dr, dl, 256, mc)
    b = orc.match_features(dr, dl, 256, mc)
    assert len(a) > 400 and np.array_equal(a, b)
    # perturbed descriptors: ratio test and multi-probe paths get exercised
    rng = np.random.default_rng(3)
    noisy = dr.copy()
    flips = rng.integers(0, 64, size=(len(dr), 6))
    for i, f in enumerate(flips):
        for b_ in f:
            noisy[i, b_ // 64 * 0 + (b_ % 4)] ^= np.uint64(1) << np.uint64(b_)
    for t_probes, L, k in ((16, 4, 16), (40, 6, 12), (1, 1, 20)):
        mc2 = params.matching
        mc2.t_probes, mc2.tables, mc2.bits = t_probes, L, k
        a = lp.match_features(noisy, dl, 256, mc2)
        b = orc.match_features(noisy, dl, 256, mc2)
        assert np.array_equal(a, b), (t_probes, L, k)
    mc2.t_probes, mc2.tables, mc2.bits = 16, 4, 16


def test_match_features_large_sets(lp, orc, params):
    """More accepted matches than k_match_finalize's shared-memory rank
    placement holds (> 16K): the radix-sorted finalize path (match.cu,
    prims.cuh). 20K train descriptors, 20K queries that are noisy copies."""
    rng = np.random.default_rng(11)
    n = 20_000
    train = rng.integers(0, 2**63, size=(n, 8), dtype=np.uint64)
    train[:, 4:] &= ~train[:, :4]  # ternary planes disjoint
    query = train.copy()
    flips = rng.integers(0, 256, size=(n, 3))
    for i, f in enumerate(flips):
        for b_ in f:
            query[i, b_ // 64] ^= np.uint64(1) << np.uint64(b_ % 64)
    query[:, 4:] &= ~query[:, :4]
    perm = rng.permutation(n)
    query = query[perm]
    mc = params.matching
    a = lp.match_features(query, train, 256, mc)
    b = orc.match_features(query, train, 256, mc)
    assert len(a) > 16_384 and np.array_equal(a, b)


def test_descriptor_distances(lp, orc):
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**63, size=(50, 8), dtype=np.uint64)
    b = rng.integers(0, 2**63, size=(50, 8), dtype=np.uint64)
    assert np.array_equal(lp.descriptor_distances(a, b, 256), orc.descriptor_distances(a, b, 256))


# ---------------------------------------------------------------- homography
def test_dlt(lp, orc):
    for seed in range(4):
        src, dst, q = prosac_data(seed, n=200)
        corr = orc.corr_array(src, dst, q)
        for n in (4, 5, 70, 200):
            a = lp.dlt_homography(corr[:n])
            b = orc.dlt_homography(corr[:n])
            assert frob_rel(a, b) < 1e-4
            assert np.array_equal(a, b), (seed, n, frob_rel(a, b))


@pytest.mark.parametrize("seed", [0, 1, 7, 1234])
def test_prosac(lp, orc, seed):
    src, dst, q = prosac_data(seed + 3, n=300, inlier_frac=0.5, noise=1.0)
    corr = orc.corr_array(src, dst, q)
    for sampling in (0, 1):
        pc = orc.default_params().prosac
        pc.seed = seed
        pc.sampling = sampling
        a = lp.prosac_homography(corr, pc, trace=True)
        b = orc.prosac_homography(corr, pc, trace=True)
        assert a["iterations"] == b["iterations"]
        assert np.array_equal(a["pool"], b["pool"])
        assert np.array_equal(a["samples"], b["samples"])
        assert frob_rel(a["model"], b["model"]) < 1e-4
        assert np.array_equal(a["model"], b["model"])
        assert np.array_equal(a["mask"], b["mask"]) and a["inlier_count"] == b["inlier_count"]


def test_prosac_errors(lp, orc):
    from paper_1810_03988_b200 import LorbError
    pc = orc.default_params().prosac
    few = orc.corr_array([[0, 0]] * 3, [[0, 0]] * 3, [1, 1, 1])
    for o in (lp, orc):
        with pytest.raises(LorbError) as e:
            o.prosac_homography(few, pc)
        assert e.value.name == "InsufficientMatches"
    line = orc.corr_array([[i, 2 * i] for i in range(20)], [[i, 2 * i] for i in range(20)], [1] * 20)
    names = []
    for o in (lp, orc):
        with pytest.raises(LorbError) as e:
            o.prosac_homography(line, pc)
        names.append(e.value.name)
    assert names == ["NoModelFound", "NoModelFound"]


# ---------------------------------------------------------------- compositor
def _scene(orc):
    l, r, th = orc.planted_pair(200, 150, 0.25, 8)
    homs = [np.eye(3), np.array([[1, 0, th[2]], [0, 1, 0], [0, 0, 1.0]]) @ np.array(
        [[1, 0.003, 0.6], [-0.002, 1, 0.25], [1e-5, 0, 1.0]])]
    cv, _ = orc.compute_canvas([(200, 150), (200, 150)], homs)
    return l, r, homs, cv


def test_warp_seam(lp, orc):
    l, r, homs, cv = _scene(orc)
    for img, H in ((l, homs[0]), (r, homs[1])):
        a = lp.warp_image(img.astype(np.float32), H, cv)
        b = orc.warp_image(img.astype(np.float32), H, cv)
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    rgb = np.random.default_rng(2).uniform(0, 255, size=(150, 200, 3)).astype(np.float32)
    a = lp.warp_image(rgb, homs[1], cv)
    b = orc.warp_image(rgb, homs[1], cv)
    assert a[0].tobytes() == b[0].tobytes()
    covs = np.stack([orc.warp_image(l.astype(np.float32), homs[0], cv)[1],
                     orc.warp_image(r.astype(np.float32), homs[1], cv)[1]])
    covs[0, 40:60, 30:90] = 0  # holes: several runs per row
    assert lp.linear_seam_mask(covs).tobytes() == orc.linear_seam_mask(covs).tobytes()


def test_pyramids(lp, orc):
    rng = np.random.default_rng(5)
    for w, h in ((101, 77), (64, 64), (2, 3)):
        img = rng.uniform(0, 255, size=(h, w)).astype(np.float32)
        if w >= 2 and h >= 2:
            assert lp.downsample(img).tobytes() == orc.downsample(img).tobytes()
        for tw, th in ((2 * w, 2 * h), (2 * w + 1, 2 * h - 1)):
            assert lp.upsample(img, tw, th).tobytes() == orc.upsample(img, tw, th).tobytes()
    img = rng.uniform(0, 255, size=(77, 101)).astype(np.float32)
    for L in (1, 3, 5):
        for f in ("gaussian_pyramid", "build_laplacian"):
            a, b = getattr(lp, f)(img, L), getattr(orc, f)(img, L)
            assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b)), (f, L)
        lap = orc.build_laplacian(img, L)
        assert lp.collapse_laplacian(lap).tobytes() == orc.collapse_laplacian(lap).tobytes()


@pytest.mark.parametrize("levels", [1, 3, 4])
def test_multiband_blend(lp, orc, levels):
    l, r, homs, cv = _scene(orc)
    w0, c0 = orc.warp_image(l.astype(np.float32), homs[0], cv)
    w1, c1 = orc.warp_image(r.astype(np.float32), homs[1], cv)
    masks = orc.linear_seam_mask(np.stack([c0, c1]))
    imgs = np.stack([w0, w1])
    assert np.array_equal(lp.multiband_blend(imgs, masks, levels), orc.multiband_blend(imgs, masks, levels))


# ---------------------------------------------------------------- whole frames
def _assert_frame_equal(a, b):
    assert a["canvas"] == b["canvas"]
    for c in range(len(a["keypoints"])):
        assert np.array_equal(a["keypoints"][c], b["keypoints"][c]), c
        assert np.array_equal(a["descriptors"][c], b["descriptors"][c]), c
    for p in range(len(a["matches"])):
        assert np.array_equal(a["matches"][p], b["matches"][p]), p
    assert np.array_equal(a["homographies"], b["homographies"])
    assert np.array_equal(a["panorama"], b["panorama"])


def test_stitch_frame_cfg1(lp, orc, params):
    """BASELINE config 1: two 640x480 planted frames, L-ORB + LSH + PROSAC + blend."""
    l, r, th = orc.planted_pair(640, 480, 0.25, 42)
    a = lp.stitch_frame([l, r], params, frame_index=0)
    b = orc.stitch_frame([l, r], params, frame_index=0)
    _assert_frame_equal(a, b)
    assert abs(a["homographies"][1][0, 2] - th[2]) < 1e-6


def test_stitch_sequence_cfg2_small(lp, orc, params):
    """Config 2 style: sequence frames with a moving square, per-frame re-registration."""
    for t in (0, 5, 31):
        l, r = orc.sequence_frame(480, 270, t, 0.25, 42)
        _assert_frame_equal(lp.stitch_frame([l, r], params, frame_index=t),
                            orc.stitch_frame([l, r], params, frame_index=t))


def test_stitch_chain_4cam_small(lp, orc, params):
    """Config 3/4 style chain (smaller frames): 4 cameras, 6 regions, 3 pairs."""
    cams, wide, shift = chain_cameras(orc, 4, 400, 240)
    _assert_frame_equal(lp.stitch_frame(cams, params, frame_index=2),
                        orc.stitch_frame(cams, params, frame_index=2))


def test_pyramid_tma_staging_matches_cp_async(lp, orc, params, monkeypatch):
    """k_pyr_down2 stages interior boxes with TMA tensor loads (zero fill
    outside the camera window) and canvas-edge boxes with cp.async; with
    LPB_TMA=0 every box takes the cp.async path. Both panoramas must equal the
    oracle's bit for bit (1920x1080 x 4 chain: 5 pyramid levels' worth of
    interior and edge boxes)."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    cams, wide, shift = chain_cameras(orc, 4, 1920, 1080)
    want = orc.stitch_frame(cams, p, frame_index=0)
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("LPB_TMA", mode)
        rig = Rig(lp, 4, 1920, 1080, p)
        got[mode] = rig.stitch(cams, 0)["panorama"]
    assert np.array_equal(got["1"], want["panorama"])
    assert np.array_equal(got["0"], want["panorama"])


def test_rig_cache_and_device_inputs(lp, orc, params):
    """HomographyCache semantics (pipeline.hpp:259-286) and device-resident inputs."""
    import torch
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 3
    l, r, _ = orc.planted_pair(320, 240, 0.25, 42)
    rig = Rig(lp, 2, 320, 240, p)
    outs = [rig.stitch([l, r], t) for t in range(4)]
    assert [o["estimated"] for o in outs] == [True, False, False, True]
    want = orc.stitch_frame([l, r], p, frame_index=0)
    assert np.array_equal(outs[1]["panorama"], want["panorama"])
    dev = [torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()]
    o = rig.stitch(dev, 4)
    assert np.array_equal(o["panorama"], want["panorama"])


def test_full_size_4k_4cam(lp, ref, params):
    """Config 3 at full size (4 cameras x 3840x2160, canvas ~12480x2160): the
    whole frame bit-exact against the reference itself, plus size-independent
    properties: every chained homography is the planted shift (frobenius_rel
    < 1e-4) and the panorama reproduces the wide texture to +-1 LSB on >= 99%
    of the covered canvas."""
    cams, wide, shift = chain_cameras(ref, 4, 3840, 2160)
    from paper_1810_03988_b200 import Rig
    rig = Rig(lp, 4, 3840, 2160, params)
    out = rig.stitch(cams, 0, details=True)
    H = out["homographies"]
    for c in range(4):
        want = np.array([[1, 0, c * shift], [0, 1, 0], [0, 0, 1.0]])
        assert frob_rel(H[c], want) < 1e-4
    W, Hh, ox, oy = out["canvas"]
    sub = out["panorama"][-oy:-oy + 2160, -ox:-ox + wide.shape[1]].astype(int)
    assert (np.abs(sub - wide.astype(int)) <= 1).mean() >= 0.99
    assert [len(k) for k in out["keypoints"]] == [500, 1000, 1000, 500]
    ref_frame = ref.stitch_frame(cams, params, frame_index=0)
    _assert_frame_equal(out, ref_frame)


def test_errors_match_oracle(lp, orc):
    from paper_1810_03988_b200 import LorbError
    img = rand_image(32, 32, 1)
    calls = [
        lambda o: o.fast_corners(img, (0, 0, 3, 3, 0)),
        lambda o: o.harris_response(img, np.array([[2, 2]])),
        lambda o: o.upsample(np.zeros((4, 4), np.float32), 12, 8),
        lambda o: o.gaussian_pyramid(np.zeros((4, 4), np.float32), 5),
        lambda o: o.downsample(np.zeros((1, 4), np.float32)),
        lambda o: o.match_features(np.zeros((0, 8), np.uint64), np.zeros((3, 8), np.uint64), 256,
                                   o.default_params().matching),
        lambda o: o.dlt_homography(o.corr_array([[0, 0], [1, 1], [2, 2], [0, 5]],
                                                [[0, 0], [1, 1], [2, 2], [0, 5]], [1] * 4)),
    ]
    for f in calls:
        names = []
        for o in (lp, orc):
            with pytest.raises(LorbError) as e:
                f(o)
            names.append(e.value.name)
        assert names[0] == names[1], names


def test_rig_frames_in_flight(lp, orc, params):
    """lp_rig_submit / lp_rig_wait with 3 frames in flight: panoramas equal the
    synchronous path frame by frame (host and device outputs)."""
    import torch
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    frames = [orc.sequence_frame(480, 270, t, 0.25, 42) for t in range(5)]
    want = []
    ref_rig = Rig(lp, 2, 480, 270, p)
    for t, (l, r) in enumerate(frames):
        want.append(ref_rig.stitch([l, r], t)["panorama"])
    rig = Rig(lp, 2, 480, 270, p)
    cap = rig.panorama_capacity()
    host = [torch.zeros(cap, dtype=torch.uint8).pin_memory() for _ in range(5)]
    ins = [[torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory()] for l, r in frames]
    tickets = [rig.submit([a.data_ptr(), b.data_ptr()], t, host[t].data_ptr(), cap) for t, (a, b) in enumerate(ins)]
    for t, tk in enumerate(tickets):
        W, H, _, _ = rig.wait(tk)
        got = host[t][:W * H].numpy().reshape(H, W)
        assert np.array_equal(got, want[t]), t


def test_rig_frames_in_flight_with_details(lp, orc):
    """lp_rig_submit_frame / lp_rig_wait_frame: 3 frames in flight, each
    re-registering (refresh 1, moving square), every frame's keypoints,
    descriptors, matches, homographies and panorama equal to the synchronous
    details of the same frame and to the oracle's."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1
    frames = [orc.sequence_frame(480, 270, t, 0.25, 42) for t in range(7)]
    rig = Rig(lp, 2, 480, 270, p)
    inflight, got = [], {}
    for t, (l, r) in enumerate(frames):
        inflight.append((t, rig.submit_frame([l, r], t)))
        if len(inflight) == 3:
            t0, h = inflight.pop(0)
            got[t0] = rig.wait_frame(h)
    for t0, h in inflight:
        got[t0] = rig.wait_frame(h)
    for t, (l, r) in enumerate(frames):
        want = orc.stitch_frame([l, r], p, frame_index=t)
        g = got[t]
        assert g["estimated"]
        assert g["canvas"] == want["canvas"], t
        for c in range(2):
            assert np.array_equal(g["keypoints"][c], want["keypoints"][c]), (t, c)
            assert np.array_equal(g["descriptors"][c], want["descriptors"][c]), (t, c)
        assert np.array_equal(g["matches"][0], want["matches"][0]), t
        assert np.array_equal(g["homographies"], want["homographies"]), t
        assert np.array_equal(g["panorama"], want["panorama"]), t
        assert g["stage_ms"][3] > 0


@pytest.mark.parametrize("in_flight", [1, 3])
def test_async_reregistration_geometry_changes(lp, orc, in_flight):
    """Once a homography set is cached, a refresh frame's verdict, inverse maps
    and geometry check come from the device (k_geom) and the host harvests
    them later. Frames here alternate between two planted overlaps, so the
    canvas and the windows move between frames and the host must compose
    those frames again on their own geometry (repair), with up to 3 frames
    in flight; every panorama, homography and match list equals the
    oracle's for that frame."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1
    overlaps = [0.25, 0.35, 0.35, 0.25, 0.30, 0.30, 0.25]
    frames = [orc.planted_pair(480, 270, ov, 7)[:2] for ov in overlaps]
    rig = Rig(lp, 2, 480, 270, p)
    got, inflight = {}, []
    for t, (l, r) in enumerate(frames):
        inflight.append((t, rig.submit_frame([l, r], t)))
        if len(inflight) >= in_flight:
            t0, hnd = inflight.pop(0)
            got[t0] = rig.wait_frame(hnd)
    for t0, hnd in inflight:
        got[t0] = rig.wait_frame(hnd)
    for t, (l, r) in enumerate(frames):
        want = orc.stitch_frame([l, r], p, frame_index=t)
        g = got[t]
        assert g["canvas"] == want["canvas"], (t, g["canvas"], want["canvas"])
        assert np.array_equal(g["homographies"], want["homographies"]), t
        assert np.array_equal(g["matches"][0], want["matches"][0]), t
        assert np.array_equal(g["panorama"], want["panorama"]), t


@pytest.mark.gpu
@pytest.mark.parametrize("in_flight", [1, 3])
def test_geometry_arenas_evicted_and_revisited(lp, orc, in_flight):
    """The rig keeps the compositor arenas and graphs of its last six
    geometries (LRU). Eight planted overlaps give eight canvases: cycling
    through them evicts arenas, revisits kept ones and rebuilds evicted ones,
    with frames in flight; every frame equals the oracle's."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1
    ovs = [0.22, 0.24, 0.26, 0.28, 0.30, 0.32, 0.34, 0.36]
    order = [0, 1, 2, 3, 4, 5, 6, 7, 1, 7, 0, 4, 0, 2, 6, 6]
    pairs = {i: orc.planted_pair(480, 270, ovs[i], 11)[:2] for i in set(order)}
    rig = Rig(lp, 2, 480, 270, p)
    got, inflight = {}, []
    for t, i in enumerate(order):
        inflight.append((t, rig.submit_frame(list(pairs[i]), t)))
        if len(inflight) >= in_flight:
            t0, hnd = inflight.pop(0)
            got[t0] = rig.wait_frame(hnd)
    for t0, hnd in inflight:
        got[t0] = rig.wait_frame(hnd)
    canvases = set()
    for t, i in enumerate(order):
        want = orc.stitch_frame(list(pairs[i]), p, frame_index=t)
        g = got[t]
        canvases.add(tuple(want["canvas"]))
        assert g["canvas"] == want["canvas"], (t, g["canvas"], want["canvas"])
        assert np.array_equal(g["panorama"], want["panorama"]), t
    assert len(canvases) > 6, canvases


@pytest.mark.gpu
@pytest.mark.parametrize("in_flight", [1, 3])
def test_mask_reuse_across_cached_frames(lp, orc, in_flight):
    """Seam masks, coverage runs and the mask pyramid depend only on the
    inverse maps and windows, so frames composed on the maps of the previous
    frame reuse them (MaskState) while their image pyramids are rebuilt from
    new content. Frames here change content every frame and re-register
    every third (new maps, same or moved geometry): every panorama equals the
    oracle's for that frame."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 3
    frames = [orc.planted_pair(480, 270, 0.25 + 0.05 * (t // 3 % 2), 11 + t)[:2] for t in range(8)]
    rig = Rig(lp, 2, 480, 270, p)
    got, inflight = {}, []
    for t, (l, r) in enumerate(frames):
        inflight.append((t, rig.submit_frame([l, r], t)))
        if len(inflight) >= in_flight:
            t0, hnd = inflight.pop(0)
            got[t0] = rig.wait_frame(hnd)
    for t0, hnd in inflight:
        got[t0] = rig.wait_frame(hnd)
    homs = None
    for t, (l, r) in enumerate(frames):
        if t % 3 == 0:  # re-registration: the whole frame from a fresh oracle engine
            want = orc.stitch_frame([l, r], p, frame_index=t)
            homs, canvas, pano = want["homographies"], want["canvas"], want["panorama"]
        else:  # the cached set: warp_blend (pipeline.hpp:499-521) with the oracle's primitives
            canvas, _ = orc.compute_canvas([(480, 270)] * 2, homs)
            warped = [orc.warp_image(img.astype(np.float32), homs[c], canvas) for c, img in enumerate((l, r))]
            masks = orc.linear_seam_mask(np.stack([cv for _, cv in warped]))
            pano = orc.multiband_blend(np.stack([wi for wi, _ in warped]), masks, p.blend_levels)
        g = got[t]
        assert g["canvas"] == canvas, (t, g["canvas"], canvas)
        assert np.array_equal(g["homographies"], homs), t
        assert np.array_equal(g["panorama"], pano), t


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,ncams,overlap", [(333, 251, 2, 0.3), (257, 190, 3, 0.3), (641, 479, 3, 0.25)])
def test_odd_frame_sizes_through_the_rig(lp, orc, w, h, ncams, overlap):
    """Frame sizes that are not multiples of the compositor's alignment (the
    generic blend kernel at some levels, cp.async staging at canvas edges,
    ragged last tiles) through the rig with 3 frames in flight; the cached
    frames reuse their seam masks. Every frame against the oracle."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    cams, _, _ = chain_cameras(orc, ncams, w, h, overlap, 11)
    want = orc.stitch_frame(cams, p, frame_index=0)
    rig = Rig(lp, ncams, w, h, p)
    hs = [rig.submit_frame(list(cams), t) for t in range(3)]
    for hnd in hs:
        g = rig.wait_frame(hnd)
        assert g["canvas"] == want["canvas"]
        assert np.array_equal(g["homographies"], want["homographies"])
        for c in range(ncams):
            assert np.array_equal(g["keypoints"][c], want["keypoints"][c]), c
        assert np.array_equal(g["panorama"], want["panorama"])


def _ref_sequence(ref, frames, p, cameras=None):
    """The reference's own StitchEngine (Serial) over the frame sequence
    (over a RigLayout when `cameras` are given): every frame's composite, or
    None where the engine dropped it."""
    import ctypes as C
    nf, ncams = len(frames), len(frames[0])
    h, w = frames[0][0].shape
    flat = [np.ascontiguousarray(im) for fr in frames for im in fr]
    arr = (C.c_void_p * len(flat))(*[im.ctypes.data for im in flat])
    stride = 64 * ncams * w * h  # room for canvases far beyond BufferPool's ncams x w x 2h
    panos = np.zeros((nf, stride), np.uint8)
    dims = np.zeros(2 * nf, np.int32)
    dropped = np.zeros(nf, np.int32)
    if cameras is None:
        fn = ref.lib.ref_run_sequence
        fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t,
                       C.c_void_p, C.c_void_p]
        st = fn(ncams, w, h, C.byref(p), arr, nf, panos.ctypes.data, stride, dims.ctypes.data,
                dropped.ctypes.data)
    else:
        fn = ref.lib.ref_run_sequence_layout
        fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                       C.c_size_t, C.c_void_p, C.c_void_p]
        cams = ref.cameras(cameras)
        st = fn(ncams, w, h, cams, C.byref(p), arr, nf, panos.ctypes.data, stride, dims.ctypes.data,
                dropped.ctypes.data)
    assert st == 0, ref.lib.ref_last_error().decode()
    out = []
    for f in range(nf):
        if dropped[f]:
            out.append(None)
        else:
            cw, ch = int(dims[2 * f]), int(dims[2 * f + 1])
            out.append(panos[f, :cw * ch].reshape(ch, cw))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(int(os.environ.get("LPB_SOAK_CASES", "12"))))
def test_randomised_rig_sequences_vs_reference_engine(lp, ref, case):
    """Soak against the reference's own StitchEngine run over the same frame
    sequence (oracle/_ref, Serial mode): random frame size, camera count,
    overlap, refresh interval and frames in flight; the scene's overlap
    changes every other frame, so re-registrations move the canvas (repairs),
    estimates fail on some frames (the reference drops those without a cache
    and falls back to the cache with one), and cached frames keep or rebuild
    their arenas and seam masks. Every panorama and every drop must match."""
    from paper_1810_03988_b200 import Rig, abi
    rng = np.random.default_rng(1000 + case)
    # LPB_SOAK_BIG=1: frames up to 1280 x 720 and up to 4 cameras (slower reference)
    big = os.environ.get("LPB_SOAK_BIG") == "1"
    w, h = (int(rng.integers(600, 1280)), int(rng.integers(400, 720))) if big else \
        (int(rng.integers(200, 520)), int(rng.integers(160, 360)))
    ncams = int(rng.integers(2, 5 if big else 4))
    refresh = int(rng.choice([1, 2, 3, 1 << 30]))
    in_flight = int(rng.integers(1, 4))
    ovs = [float(rng.uniform(0.25, 0.4)), float(rng.uniform(0.25, 0.4))]
    p = ref.default_params()
    p.seed = p.matching.seed = 42 + case
    p.homography_refresh = refresh
    frames = [chain_cameras(ref, ncams, w, h, ovs[(t // 2) % 2], 50 + case * 10 + t)[0] for t in range(8)]
    want = _ref_sequence(ref, frames, p)
    rig = Rig(lp, ncams, w, h, p)
    got, pending = {}, []

    def land(t0, hnd):
        try:
            got[t0] = rig.wait_frame(hnd)["panorama"]
        except abi.LorbError:
            got[t0] = None

    for t, cams in enumerate(frames):
        try:
            pending.append((t, rig.submit_frame(list(cams), t)))
        except abi.LorbError:
            got[t] = None
        if len(pending) >= in_flight:
            land(*pending.pop(0))
    for t0, hnd in pending:
        land(t0, hnd)
    for t in range(len(frames)):
        ctx = (case, w, h, ncams, refresh, in_flight, t)
        if want[t] is None:
            assert got[t] is None, ctx
        else:
            assert got[t] is not None, ctx
            assert np.array_equal(got[t], want[t]), ctx


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(int(os.environ.get("LPB_SOAK_CASES", "12"))))
def test_randomised_parameters_vs_reference_engine(lp, ref, case):
    """Soak over the parameter space (FAST threshold and arc, Harris sigma
    and threshold, top_n, descriptor length, blur sigma, LSH tables / bits /
    probes, ratio, PROSAC threshold / iterations / sampling, blend levels,
    overlap fraction), each case a 5-frame sequence through the rig and
    through the reference's own StitchEngine: every panorama and every drop
    equal, and a parameter set the reference rejects is rejected by the rig
    with the same status."""
    from paper_1810_03988_b200 import Rig, abi
    rng = np.random.default_rng(5000 + case)
    w, h = int(rng.integers(240, 480)), int(rng.integers(180, 320))
    ncams = int(rng.integers(2, 4))
    p = ref.default_params()
    p.seed = p.matching.seed = int(rng.integers(1, 1 << 30))
    e = p.extraction
    e.fast_threshold = int(rng.integers(10, 40))
    e.fast_arc = int(rng.choice([9, 10, 12]))
    e.harris_sigma = float(rng.choice([0.8, 1.0, 1.4, 2.0]))
    e.top_n = int(rng.choice([100, 200, 500, 800]))
    e.n_d = int(rng.choice([256, 512]))
    e.brief_blur_sigma = float(rng.choice([1.5, 2.0, 3.0]))
    m = p.matching
    m.tables = int(rng.integers(2, 8))
    m.bits = int(rng.choice([12, 16, 20]))
    m.t_probes = int(rng.integers(0, 3))
    m.ratio = float(rng.uniform(0.7, 0.9))
    pr = p.prosac
    pr.threshold_px = float(rng.choice([2.0, 3.0, 4.0]))
    pr.max_iter = int(rng.choice([200, 1000, 2000]))
    pr.sampling = int(rng.integers(0, 2))
    p.blend_levels = int(rng.integers(1, 6))
    p.homography_refresh = int(rng.choice([1, 2, 1 << 30]))
    ov = float(rng.uniform(0.25, 0.4))
    p.overlap_fraction = ov
    frames = [chain_cameras(ref, ncams, w, h, ov, 70 + case * 10 + t)[0] for t in range(5)]
    try:
        want = _ref_sequence(ref, frames, p)
    except AssertionError as err:  # the reference rejected the parameters
        with pytest.raises(abi.LorbError):
            rig = Rig(lp, ncams, w, h, p)
            rig.wait_frame(rig.submit_frame(list(frames[0]), 0))
        return
    try:
        rig = Rig(lp, ncams, w, h, p)
    except abi.LorbError as err:
        # the C-ABI rejects at creation what the reference's engine rejects
        # in a stage of every frame (each frame dropped; the drop-in
        # pipeline.hpp creates the rig inside its stage and drops them too)
        assert err.name == "BadParams" and all(x is None for x in want), (case, str(err))
        return
    for t, cams in enumerate(frames):
        try:
            g = rig.wait_frame(rig.submit_frame(list(cams), t))["panorama"]
        except abi.LorbError:
            g = None
        ctx = (case, w, h, ncams, t)
        if want[t] is None:
            assert g is None, ctx
        else:
            assert g is not None, ctx
            assert np.array_equal(g, want[t]), ctx


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(int(os.environ.get("LPB_SOAK_CASES", "12")) // 2))
def test_randomised_layout_sequences_vs_reference_engine(lp, ref, case):
    """Soak over RigLayouts: per-camera pre-transforms (small rotations,
    shears, perspective terms) and crops, stitched through lp_rig_create_layout
    (stage_rectify_crop on ingest) and through the reference's own engine over
    the same 5-frame sequence; every panorama and every drop equal."""
    from paper_1810_03988_b200 import Rig, abi
    rng = np.random.default_rng(9000 + case)
    w, h = int(rng.integers(260, 520)), int(rng.integers(200, 360))
    ncams = int(rng.integers(2, 4))
    p = ref.default_params()
    p.seed = p.matching.seed = 42 + case
    p.homography_refresh = int(rng.choice([1, 2, 1 << 30]))
    ov = float(rng.uniform(0.3, 0.4))
    p.overlap_fraction = ov
    specs = []
    cw, ch = w - int(rng.integers(8, 24)), h - int(rng.integers(8, 24))  # one rectified size for all cameras
    for c in range(ncams):
        t = np.deg2rad(float(rng.uniform(-2.0, 2.0)))
        co, si = np.cos(t), np.sin(t)
        H = np.array([[co, -si, w / 2 - co * w / 2 + si * h / 2 + rng.uniform(-1, 1)],
                      [si, co, h / 2 - si * w / 2 - co * h / 2 + rng.uniform(-1, 1)],
                      [rng.uniform(-2e-5, 2e-5), rng.uniform(-2e-5, 2e-5), 1.0]])
        x0, y0 = int(rng.integers(0, w - cw + 1)), int(rng.integers(0, h - ch + 1))
        specs.append((H if rng.random() < 0.7 else None, (x0, y0, x0 + cw, y0 + ch)))
    frames = [chain_cameras(ref, ncams, w, h, ov, 90 + case * 10 + t)[0] for t in range(5)]
    want = _ref_sequence(ref, frames, p, cameras=specs)
    rig = Rig(lp, ncams, w, h, p, cameras=specs)
    for t, cams in enumerate(frames):
        try:
            g = rig.wait_frame(rig.submit_frame(list(cams), t))["panorama"]
        except abi.LorbError:
            g = None
        ctx = (case, w, h, ncams, t)
        if want[t] is None:
            assert g is None, ctx
        else:
            assert g is not None, ctx
            assert np.array_equal(g, want[t]), ctx


@pytest.mark.gpu
def test_rig_reset_is_a_fresh_engine(lp, orc):
    """lp_rig_reset (the drop-in engine's rig pool): after a reset the rig
    forgets its HomographyCache, so frames of another scene estimate again
    from frame 0 and equal the oracle's fresh engine, with up to 3 in flight."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    first = orc.planted_pair(480, 270, 0.25, 7)[:2]
    second = orc.planted_pair(480, 270, 0.35, 8)[:2]
    rig = Rig(lp, 2, 480, 270, p)
    hs = [rig.submit_frame(list(first), t) for t in range(3)]
    for h in hs:
        rig.wait_frame(h)
    rig.reset()
    want = orc.stitch_frame(list(second), p, frame_index=0)
    got = [rig.wait_frame(rig.submit_frame(list(second), t)) for t in range(2)]
    for g in got:
        assert g["canvas"] == want["canvas"]
        assert np.array_equal(g["homographies"], want["homographies"])
        assert np.array_equal(g["panorama"], want["panorama"])


@pytest.mark.gpu
def test_concurrent_rigs_threads(lp, orc):
    """Independent rigs on one context, driven from host threads (the config-5
    shape): each rig has its own stage stream, so their frames overlap on the
    device; every panorama must equal the oracle's for that rig's input."""
    import threading

    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    nrig, frames = 6, 3
    inputs = [orc.planted_pair(320, 240, 0.25, 100 + i)[:2] for i in range(nrig)]
    want = [orc.stitch_frame(list(inputs[i]), p, frame_index=0)["panorama"] for i in range(nrig)]
    rigs = [Rig(lp, 2, 320, 240, p) for _ in range(nrig)]
    got = [[None] * frames for _ in range(nrig)]
    errs = []

    def run(i):
        try:
            for f in range(frames):
                got[i][f] = rigs[i].stitch(list(inputs[i]), f)["panorama"]
        except Exception as e:  # surfaced below
            errs.append(e)
    ths = [threading.Thread(target=run, args=(i,)) for i in range(nrig)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for i in range(nrig):
        for f in range(frames):
            assert np.array_equal(got[i][f], want[i]), (i, f)


def test_rig_graph_replay_matches_direct(lp, orc):
    """The compositor chain replayed as a CUDA graph (default) gives the same
    panoramas as individually launched kernels, across slot reuse."""
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    frames = [orc.sequence_frame(400, 300, t, 0.25, 42) for t in range(7)]
    direct = Rig(lp, 2, 400, 300, p)
    direct.set_graphs(False)
    graph = Rig(lp, 2, 400, 300, p)
    for t, (l, r) in enumerate(frames):
        a = direct.stitch([l, r], t)["panorama"]
        b = graph.stitch([l, r], t)["panorama"]
        assert np.array_equal(a, b), t


def test_rig_nondefault_params_generic_paths(lp, orc):
    """A 3-camera rig with non-default parameters: Harris sigma 1.5 and FAST
    arc 10 (generic detect kernel), n_d 512 and blur sigma 3 (generic
    describe), top_n 300, 6 blend levels (levels 5+ take the generic blend
    kernel) and an odd frame size, bit-exact against the oracle."""
    p = orc.default_params()
    p.seed = p.matching.seed = 7
    p.extraction.harris_sigma = 1.5
    p.extraction.fast_arc = 10
    p.extraction.n_d = 512
    p.extraction.brief_blur_sigma = 3.0
    p.extraction.top_n = 300
    p.blend_levels = 6
    cams, _, _ = chain_cameras(orc, 3, 501, 397, 0.25, 11)
    got = lp.stitch_frame(cams, p, frame_index=0)
    want = orc.stitch_frame(cams, p, frame_index=0)
    assert got["canvas"] == want["canvas"]
    for c in range(3):
        assert np.array_equal(got["keypoints"][c], want["keypoints"][c]), c
        assert np.array_equal(got["descriptors"][c], want["descriptors"][c]), c
    for q in range(2):
        assert np.array_equal(got["matches"][q], want["matches"][q]), q
    assert np.array_equal(got["homographies"], want["homographies"])
    assert np.array_equal(got["panorama"], want["panorama"])


def test_rig_refresh_every_frame_graph_updates(lp, orc):
    """Re-registration on every frame with device-resident inputs (estimate on
    the feature stream) and CUDA graphs: homographies that change below a
    pixel of canvas patch the k_warp node in place, a different overlap moves
    the canvas (graph recapture + in-place update); every panorama equals the
    oracle's stitch_frame for that frame and the direct-launch rig's."""
    import torch
    from paper_1810_03988_b200 import Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1
    frames = [orc.sequence_frame(400, 300, t, 0.25, 42) for t in range(5)]
    l2, r2, _ = orc.planted_pair(400, 300, 0.3, 7)
    frames += [(l2, r2)] + [orc.sequence_frame(400, 300, t, 0.25, 42) for t in range(5, 8)]
    direct = Rig(lp, 2, 400, 300, p)
    direct.set_graphs(False)
    graph = Rig(lp, 2, 400, 300, p)
    for t, (l, r) in enumerate(frames):
        want = orc.stitch_frame([l, r], p, frame_index=t)["panorama"]
        a = direct.stitch([l, r], t)["panorama"]
        dev = [torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()]
        b = graph.stitch(dev, t)["panorama"]
        assert np.array_equal(a, want), t
        assert np.array_equal(b, want), t


def test_prosac_single_cta_path_matches(tmp_path):
    """PROSAC's one-CTA launch (LPB_PROSAC_CLUSTER=0, also the in-kernel
    fallback for very large correspondence sets) against the oracle, in a
    fresh process (the launch mode is read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys
sys.path.insert(0, %r)
import numpy as np
from oracle import Oracle
from paper_1810_03988_b200 import Lorb
from tests.golden.make_golden import prosac_data
orc, lp = Oracle("orc"), Lorb(0)
for seed in (1, 2):
    src, dst, q = prosac_data(seed + 3, n=300, inlier_frac=0.5, noise=1.0)
    corr = orc.corr_array(src, dst, q)
    pc = orc.default_params().prosac
    pc.seed = seed
    a = lp.prosac_homography(corr, pc, trace=True)
    b = orc.prosac_homography(corr, pc, trace=True)
    assert a["iterations"] == b["iterations"] and np.array_equal(a["samples"], b["samples"])
    assert np.array_equal(a["model"], b["model"]) and np.array_equal(a["mask"], b["mask"])
print("ok")
''' % root
    env = dict(os.environ, LPB_PROSAC_CLUSTER="0")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout + out.stderr


def test_rig_failed_frame_is_dropped_alone(lp, orc):
    """A device-side failure raised by one frame (per-slot status words,
    k_status_take) fails only that frame's wait(); the frames before and
    after it, in flight at the same time, complete and equal the oracle, as
    the reference engine drops one failed frame and carries on
    (pipeline.hpp run_stage -> Metrics::drops)."""
    import torch
    from paper_1810_03988_b200 import LorbError, Rig
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    frames = [orc.sequence_frame(320, 240, t, 0.25, 42) for t in range(7)]
    clean = Rig(lp, 2, 320, 240, p)
    want = [clean.stitch(list(f), t)["panorama"] for t, f in enumerate(frames)]
    assert np.array_equal(want[0], orc.stitch_frame(list(frames[0]), p, frame_index=0)["panorama"])
    rig = Rig(lp, 2, 320, 240, p)
    rig.stitch(list(frames[0]), 0)
    rig.inject_fault(3, 24)  # LP_CAPACITY_OVERFLOW on frame 3
    cap = rig.panorama_capacity()
    host = [torch.zeros(cap, dtype=torch.uint8).pin_memory() for _ in frames]
    ins = [[torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory()] for l, r in frames]
    tickets = [rig.submit([a.data_ptr(), b.data_ptr()], t, host[t].data_ptr(), cap)
               for t, (a, b) in enumerate(ins) if t > 0]
    for t, tk in zip(range(1, 7), tickets):
        if t == 3:
            with pytest.raises(LorbError) as e:
                rig.wait(tk)
            assert e.value.name == "CapacityOverflow"
            continue
        W, H, _, _ = rig.wait(tk)
        got = host[t][:W * H].numpy().reshape(H, W)
        assert np.array_equal(got, want[t]), t
    # and the rig keeps working synchronously afterwards
    out = rig.stitch(list(frames[5]), 8)
    assert np.array_equal(out["panorama"], want[5])


def test_rig_feature_fault_survives_repair(lp, orc):
    """A frame whose feature stage fails and whose device verdict also moves
    the canvas (so the rig recomposes it: repair) still fails at its wait():
    the recomposition's status take must not overwrite the feature stage's
    error with the recomposition's clean status. Inputs: the bench's config-1
    style frame sets (the reference's synth::texture cut into two cameras, a
    moving square per set), re-registered every frame, whose estimates give
    canvases a pixel apart."""
    from paper_1810_03988_b200 import LorbError, Rig
    from paper_1810_03988_b200.lib import synth_texture
    w, h, n = 640, 480, 16
    shift = int(np.floor(w * 0.75 + 0.5))
    wide = synth_texture(w + shift, h, 42)
    size = max(4, h // 16)
    frames = []
    for s in range(8):
        cams = [np.ascontiguousarray(wide[:, c * shift:c * shift + w]).copy() for c in range(2)]
        px, py = (s * 7 * 37) % (w - size), (s * 3 * 37) % (h - size)
        for c in range(2):
            x0 = px - c * shift
            if -size < x0 < w:
                cams[c][py:py + size, max(0, x0):min(w, x0 + size)] = 255
        frames.append(cams)
    p = orc.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1
    clean = Rig(lp, 2, w, h, p)
    canv = [clean.stitch(list(frames[t % 8]), t)["canvas"] for t in range(n)]
    moved = [t for t in range(2, n) if canv[t] != canv[t - 1]]
    if not moved:
        pytest.skip("no canvas jitter between these estimates")
    bad = moved[0]
    rig = Rig(lp, 2, w, h, p)
    for t in range(bad):
        assert rig.stitch(list(frames[t % 8]), t)["canvas"] == canv[t]
    rig.inject_fault(bad, 10)  # LP_WINDOW_OUT_OF_BOUNDS in the feature stage of a repaired frame
    with pytest.raises(LorbError) as e:
        rig.stitch(list(frames[bad % 8]), bad)
    assert e.value.name == "WindowOutOfBounds"
    # the frames after it are unaffected
    for t in range(bad + 1, min(bad + 4, n)):
        assert rig.stitch(list(frames[t % 8]), t)["canvas"] == canv[t]
