"""Pin the C restatement oracle (oracle/lorb_oracle.c) to the reference.

Fixtures: tests/golden/golden.npz, produced by tests/golden/make_golden.py from
the unmodified reference compiled in place (oracle/_ref). Every array must be
bit-identical: features, descriptors, LSH bit positions and probe masks,
matches, PROSAC traces/models, warp/seam/pyramid/blend rasters and a whole
frame's panorama. CPU only."""
import os

import numpy as np
import pytest

from tests.golden.make_golden import cases, prosac_data, rand_u8

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="module")
def orc_cases(orc):
    return cases(orc)


def test_golden_keys_complete(golden, orc_cases):
    assert set(golden) == set(orc_cases)


@pytest.mark.parametrize("key", sorted(dict(np.load(GOLDEN)).keys()))
def test_restatement_matches_reference_golden(golden, orc_cases, key):
    want, got = golden[key], np.asarray(orc_cases[key])
    assert want.shape == got.shape, key
    assert want.dtype == got.dtype or want.size == 0, key
    # bit-identical, floats compared through their bytes
    assert want.tobytes() == got.tobytes(), key


def test_known_answers(orc):
    """KATs the reference's own tests state (test_matchlsh.cpp:99-123)."""
    assert list(orc.probe_sequence(2, 4)) == [0, 1, 2, 3]
    assert list(orc.probe_sequence(16, 1)) == [0]
    p16 = orc.probe_sequence(16, 16)
    assert list(p16) == [0] + [1 << i for i in range(15)]  # bit 15 never flipped
    # seed 42 table 0 bit positions
    assert list(orc.lsh_bit_positions(256, 4, 16, 42)[0]) == [
        386, 327, 385, 72, 462, 52, 296, 195, 146, 205, 16, 273, 354, 331, 425, 485]
    # seed 42 pattern starts (-3,3)-(2,-4)
    assert list(orc.brief_pattern(256, 15, 42)[0]) == [-3, 3, 2, -4]
    k = orc.gaussian_kernel(2.0)
    assert len(k) == 13 and abs(k[6] - 0.199675635) < 1e-8


def test_live_against_reference(ref, orc):
    """Extra random cases against the reference itself (build container only)."""
    for s in range(6):
        img = rand_u8(96, 80, 100 + s)
        for arc in (9, 10, 16):
            a = ref.fast_corners(img, (4, 6, 90, 77, 0), 10 + s, arc)
            b = orc.fast_corners(img, (4, 6, 90, 77, 0), 10 + s, arc)
            assert np.array_equal(a, b)
    src, dst, q = prosac_data(5, n=300, inlier_frac=0.4, noise=1.0)
    corr = ref.corr_array(src, dst, q)
    for seed in (0, 1, 99):
        pc = ref.default_params().prosac
        pc.seed = seed
        a = ref.prosac_homography(corr, pc, trace=True)
        b = orc.prosac_homography(corr, pc, trace=True)
        assert a["iterations"] == b["iterations"]
        assert np.array_equal(a["samples"], b["samples"])
        assert np.array_equal(a["model"], b["model"])
        assert np.array_equal(a["mask"], b["mask"])
    pc.sampling = 1  # Uniform
    a = ref.prosac_homography(corr, pc, trace=True)
    b = orc.prosac_homography(corr, pc, trace=True)
    assert np.array_equal(a["samples"], b["samples"]) and np.array_equal(a["model"], b["model"])


def test_live_frame_sequence_against_reference(ref, orc, params):
    """cfg2-style sequence frames (moving square), smaller frames."""
    for t in (0, 7):
        l, r = ref.sequence_frame(320, 180, t, 0.25, 42)
        a = ref.stitch_frame([l, r], params, frame_index=t)
        b = orc.stitch_frame([l, r], params, frame_index=t)
        assert a["canvas"] == b["canvas"]
        assert np.array_equal(a["homographies"], b["homographies"])
        assert np.array_equal(a["panorama"], b["panorama"])
        for c in range(2):
            assert np.array_equal(a["keypoints"][c], b["keypoints"][c])
            assert np.array_equal(a["descriptors"][c], b["descriptors"][c])
        assert np.array_equal(a["matches"][0], b["matches"][0])


def test_error_codes_match_reference(ref, orc):
    from paper_1810_03988_b200.abi import LorbError
    img = rand_u8(32, 32, 1)
    calls = [
        lambda o: o.fast_corners(img, (0, 0, 3, 3, 0)),                  # RegionTooSmall
        lambda o: o.harris_response(img, np.array([[2, 2]])),            # WindowOutOfBounds
        lambda o: o.upsample(np.zeros((4, 4), np.float32), 12, 8),       # BadTargetDims
        lambda o: o.gaussian_pyramid(np.zeros((4, 4), np.float32), 5),   # TooManyLevels
        lambda o: o.downsample(np.zeros((1, 4), np.float32)),            # ImageTooSmall
        lambda o: o.probe_sequence(2, 5),                                # TooManyProbes
        lambda o: o.dlt_homography(o.corr_array([[0, 0]] * 3, [[0, 0]] * 3, [1, 1, 1])),
        lambda o: o.dlt_homography(o.corr_array([[0, 0], [1, 1], [2, 2], [0, 5]],
                                                [[0, 0], [1, 1], [2, 2], [0, 5]], [1] * 4)),
    ]
    for f in calls:
        names = []
        for o in (ref, orc):
            with pytest.raises(LorbError) as e:
                f(o)
            names.append(e.value.name)
        assert names[0] == names[1], names
