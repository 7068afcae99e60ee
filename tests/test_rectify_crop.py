"""stage_rectify_crop (pipeline.hpp:391-417, §8(f) row 2): per-camera
pre-transform (warp_image onto the camera's own canvas + to_u8_image) and
crop, then the whole engine over a RigLayout.

CPU: the plain-C restatement (orc_rectify_crop) against the reference itself
(oracle/_ref) byte for byte, plus the reference's error behaviour.
GPU: the CUDA path (lp_rectify_crop, lp_rig_create_layout) against the
reference on the same inputs: rectified frames, keypoints, descriptors,
matches, homographies and panorama bit-exact."""
import numpy as np
import pytest

from paper_1810_03988_b200.abi import LorbError
from tests.conftest import rand_image


def rot(deg, cx, cy, tx=0.0, ty=0.0):
    t = np.deg2rad(deg)
    c, s = np.cos(t), np.sin(t)
    return np.array([[c, -s, cx - c * cx + s * cy + tx], [s, c, cy - s * cx - c * cy + ty], [0, 0, 1]])


def cases(w, h):
    return [
        [(None, None), (None, None)],                                     # identity layout
        [(None, (5, 7, w - 9, h - 4)), (None, (3, 2, w - 11, h - 9))],   # crops only
        [(rot(1.5, w / 2, h / 2), None), (np.diag([1.0, 1.0, 1.0]), None)],
        [(rot(-3.0, w / 3, h / 2, 0.37, -1.2), (10, 10, w - 10, h - 12)),
         (np.array([[1.01, 0.002, -2.5], [-0.003, 0.995, 1.25], [1e-5, -2e-5, 1.0]]), (0, 4, w - 20, h - 8))],
    ]


def test_rectify_crop_oracle_matches_reference(orc, ref):
    w, h = 160, 120
    imgs = [rand_image(w, h, 1), orc.texture(w, h, 7)]
    for specs in cases(w, h):
        a = orc.rectify_crop(imgs, specs)
        b = ref.rectify_crop(imgs, specs)
        for x, y in zip(a, b):
            assert x.shape == y.shape and np.array_equal(x, y)


def test_rectify_crop_errors(orc, ref):
    w, h = 64, 48
    imgs = [rand_image(w, h, 2)]
    for o in (orc, ref):
        with pytest.raises(LorbError) as e:
            o.rectify_crop(imgs, [(None, (0, 0, w + 1, h))])
        assert e.value.name == "BadParams"
        with pytest.raises(LorbError) as e:
            o.rectify_crop(imgs, [(np.zeros((3, 3)), None)])
        assert e.value.name == "SingularHomography"


@pytest.mark.gpu
def test_rectify_crop_gpu(lp, ref):
    for w, h, seed in ((160, 120, 3), (641, 479, 4)):
        imgs = [rand_image(w, h, seed), ref.texture(w, h, seed + 1)]
        for specs in cases(w, h):
            a = lp.rectify_crop(imgs, specs)
            b = ref.rectify_crop(imgs, specs)
            for x, y in zip(a, b):
                assert x.shape == y.shape and np.array_equal(x, y)


@pytest.mark.gpu
def test_rectify_crop_gpu_errors(lp):
    imgs = [rand_image(64, 48, 2)]
    with pytest.raises(LorbError) as e:
        lp.rectify_crop(imgs, [(None, (0, 0, 65, 48))])
    assert e.value.name == "BadParams"
    with pytest.raises(LorbError) as e:
        lp.rectify_crop(imgs, [(np.zeros((3, 3)), None)])
    assert e.value.name == "SingularHomography"


@pytest.mark.gpu
def test_stitch_frame_layout_gpu(lp, ref, params):
    """Config-1 scene through a RigLayout: sub-pixel rectification of the
    right camera and a shared crop, bit-exact against the reference engine."""
    left, right, _ = ref.planted_pair(640, 480, 0.25, 42)
    specs = [(None, (4, 6, 632, 470)),
             (np.array([[1.0, 0.0, 0.25], [0.0, 1.0, -0.5], [0.0, 0.0, 1.0]]), (4, 6, 632, 470))]
    got = lp.stitch_frame([left, right], params, frame_index=0, cameras=specs)
    want = ref.stitch_frame([left, right], params, frame_index=0, cameras=specs)
    assert got["canvas"] == want["canvas"]
    for c in range(2):
        assert np.array_equal(got["keypoints"][c], want["keypoints"][c])
        assert np.array_equal(got["descriptors"][c], want["descriptors"][c])
    assert np.array_equal(got["matches"][0], want["matches"][0])
    assert np.array_equal(got["homographies"], want["homographies"])
    assert np.array_equal(got["panorama"], want["panorama"])
