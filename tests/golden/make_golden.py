"""Generate tests/golden/golden.npz from the REFERENCE itself.

The reference ships no golden vectors, so the fixtures are the
outputs of the unmodified reference headers compiled in place as
oracle/_ref/liblorbref.so (oracle/Makefile), on seeded inputs. The same
`cases()` runs against the C restatement in tests/test_oracle_golden.py, which
pins the restatement bit for bit before it is trusted as the GPU checker.

    python tests/golden/make_golden.py        # needs /root/reference (build box)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "golden.npz")


def rand_u8(w, h, seed):
    return np.random.default_rng(seed).integers(0, 256, size=(h, w), dtype=np.uint8)


def prosac_data(seed, n=100, inlier_frac=0.7, noise=0.5):
    """acceptance.cpp #6-style data: a planted homography, noisy inliers,
    uniform outliers, quality descending (inliers first)."""
    rng = np.random.default_rng(seed)
    H = np.array([[1.02, 0.03, 40.0], [-0.02, 0.98, -12.0], [1e-5, -2e-5, 1.0]])
    src = rng.uniform(0, 640, size=(n, 2))
    p = np.c_[src, np.ones(n)] @ H.T
    dst = p[:, :2] / p[:, 2:3]
    k = int(n * inlier_frac)
    dst[:k] += rng.normal(0, noise, size=(k, 2))
    dst[k:] = rng.uniform(0, 640, size=(n - k, 2))
    q = np.linspace(1.0, 0.5, n).astype(np.float32)
    return src, dst, q


def cases(o):
    from paper_1810_03988_b200 import abi  # noqa: F401
    g = {}
    for s in (0, 42):
        g[f"pattern_{s}"] = o.brief_pattern(256, 15, s)
        g[f"lshpos_{s}"] = o.lsh_bit_positions(256, 4, 16, s)
    for sig in (1.0, 1.5, 2.0):
        g[f"gk_{sig}"] = o.gaussian_kernel(sig)
    for k, t in ((16, 16), (2, 4), (8, 37), (4, 1)):
        g[f"probes_{k}_{t}"] = o.probe_sequence(k, t)
    g["texture"] = o.texture(64, 48, 7)
    l, r, th = o.planted_pair(160, 120, 0.25, 5)
    g["pp_left"], g["pp_right"], g["pp_h"] = l, r, th
    sl, sr = o.sequence_frame(160, 120, 9, 0.25, 5)
    g["seq_left"], g["seq_right"] = sl, sr
    # FAST / Harris / NMS / top-N on random images (acceptance.cpp #1-2 style)
    for s in range(4):
        img = rand_u8(64, 64, s)
        for arc in (9, 12, 16):
            g[f"fast_{s}_{arc}"] = o.fast_corners(img, (0, 0, 64, 64, 0), 20, arc)
        pts = g[f"fast_{s}_9"]
        pts = pts[(pts[:, 0] >= 5) & (pts[:, 0] < 59) & (pts[:, 1] >= 5) & (pts[:, 1] < 59)]
        g[f"harris_{s}"] = o.harris_response(img, pts, 0.04, 1.0)
        kp = np.zeros((len(pts), 4), np.int32)
        kp[:, :2] = pts
        kp[:, 2] = g[f"harris_{s}"].view(np.int32)
        g[f"nms_{s}"] = o.nms(kp, 1)
        g[f"topn_{s}"] = o.select_top_n(g[f"nms_{s}"], 25)
    img = np.random.default_rng(3).uniform(0, 255, size=(30, 40, 3)).astype(np.float32)
    g["blur_in"] = img
    g["blur_1.5"] = o.gaussian_blur(img, 1.5)
    # extraction on the planted pair (left strip region, lorb.hpp:388-413)
    cfg = o.default_params().extraction
    cfg.top_n = 60
    regs = o.partition_regions([(160, 120), (160, 120)], 0.25, 15)
    g["regions"] = np.array(regs, np.int32)
    kp, desc = o.extract_features(l, regs[:1], cfg, g["pattern_42"])
    g["ext_kp"], g["ext_desc"] = kp, desc
    # matching: real descriptors vs their right-camera counterparts
    kp2, desc2 = o.extract_features(r, regs[1:2], cfg, g["pattern_42"])
    mc = o.default_params().matching
    mc.seed = 42
    g["match"] = o.match_features(desc2, desc, 256, mc)
    g["dist"] = o.descriptor_distances(desc[:10], desc2[:10], 256)
    # homography
    src, dst, q = prosac_data(11)
    corr = o.corr_array(src, dst, q)
    g["dlt_all"] = o.dlt_homography(corr[:70])
    g["dlt_min"] = o.dlt_homography(corr[:4])
    pc = o.default_params().prosac
    pc.seed = 1234
    res = o.prosac_homography(corr, pc, trace=True)
    for k2, v in res.items():
        g[f"prosac_{k2}"] = np.asarray(v)
    # compositor pieces on a small two-camera scene
    f0 = l.astype(np.float32)
    homs = [np.eye(3), np.array([[1, 0, th[2]], [0, 1, 0], [0, 0, 1.0]]) @ np.array(
        [[1, 0.002, 0.4], [-0.001, 1, 0.3], [0, 0, 1.0]])]
    cv, off = o.compute_canvas([(160, 120), (160, 120)], homs)
    g["canvas"] = np.array(cv)
    w0, c0 = o.warp_image(f0, homs[0], cv)
    w1, c1 = o.warp_image(r.astype(np.float32), homs[1], cv)
    g["warp1"], g["cov1"] = w1, c1
    masks = o.linear_seam_mask(np.stack([c0, c1]))
    g["masks"] = masks
    g["down"] = o.downsample(w1)
    g["up"] = o.upsample(g["down"], w1.shape[1], w1.shape[0])
    lap = o.build_laplacian(w1, 3)
    for i, lv in enumerate(lap):
        g[f"lap_{i}"] = lv
    g["collapse"] = o.collapse_laplacian(lap)
    g["blend"] = o.multiband_blend(np.stack([w0, w1]), masks, 3)
    # one whole frame through the stage bodies (pipeline.hpp:419-521)
    p = o.default_params()
    p.seed = 42
    p.matching.seed = 42
    p.extraction.top_n = 120
    fr = o.stitch_frame([l, r], p, frame_index=3)
    g["frame_canvas"] = np.array(fr["canvas"])
    g["frame_pano"] = fr["panorama"]
    g["frame_h"] = fr["homographies"]
    for c in range(2):
        g[f"frame_kp{c}"] = fr["keypoints"][c]
        g[f"frame_desc{c}"] = fr["descriptors"][c]
    g["frame_matches"] = fr["matches"][0]
    return g


def main():
    from oracle import Oracle
    g = cases(Oracle("ref"))
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
