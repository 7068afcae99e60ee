"""symmetric_transfer_error (homography.hpp:147-152) and the PROSAC decisions
that hang on it, bit for bit against the reference.

The error is |H(s) - d| + |H^-1(d) - s| with std::hypot. The device uses a
restatement of glibc's hypot (homography.cu: glibc_hypot), not CUDA's, so an
error sitting on the 3 px inlier threshold, or two hypotheses with equal inlier
counts and error sums one ulp apart, decide the same way as on the CPU.
"""
import numpy as np
import pytest

from paper_1810_03988_b200.api import AbiWrapper

H = np.array([[1.02, 0.03, 40.0], [-0.02, 0.98, -12.0], [1e-5, -2e-5, 1.0]])


def inverse(h):
    """Homography::inverse (homography.hpp:36-48) as the reference computes it."""
    d = (h[0, 0] * (h[1, 1] * h[2, 2] - h[1, 2] * h[2, 1]) - h[0, 1] * (h[1, 0] * h[2, 2] - h[1, 2] * h[2, 0])
         + h[0, 2] * (h[1, 0] * h[2, 1] - h[1, 1] * h[2, 0]))
    inv = np.array([[(h[1, 1] * h[2, 2] - h[1, 2] * h[2, 1]) / d, (h[0, 2] * h[2, 1] - h[0, 1] * h[2, 2]) / d,
                     (h[0, 1] * h[1, 2] - h[0, 2] * h[1, 1]) / d],
                    [(h[1, 2] * h[2, 0] - h[1, 0] * h[2, 2]) / d, (h[0, 0] * h[2, 2] - h[0, 2] * h[2, 0]) / d,
                     (h[0, 2] * h[1, 0] - h[0, 0] * h[1, 2]) / d],
                    [(h[1, 0] * h[2, 1] - h[1, 1] * h[2, 0]) / d, (h[0, 1] * h[2, 0] - h[0, 0] * h[2, 1]) / d,
                     (h[0, 0] * h[1, 1] - h[0, 1] * h[1, 0]) / d]])
    if abs(inv[2, 2]) > 1e-12:
        inv = inv / inv[2, 2]
    return inv


def ste_cases(seed, n=20000):
    """Residuals of ~1.5 px per direction (errors around the 3 px threshold),
    plus exact-threshold, zero, tiny and huge residuals."""
    rng = np.random.default_rng(seed)
    src = rng.uniform(0, 3840, size=(n, 2))
    p = np.c_[src, np.ones(n)] @ H.T
    dst = p[:, :2] / p[:, 2:3]
    ang = rng.uniform(0, 2 * np.pi, n)
    r = rng.uniform(1.2, 1.8, n)
    dst += np.c_[r * np.cos(ang), r * np.sin(ang)]
    k = n // 10
    dst[:k] = p[:k, :2] / p[:k, 2:3]                       # zero forward residual
    dst[k:2 * k] += rng.normal(0, 1e-9, size=(k, 2))       # tiny
    dst[2 * k:3 * k] = rng.uniform(-1e6, 1e6, size=(k, 2))  # huge
    return src, dst


def translation_cases():
    """H a pure translation: dst = s + t + (1.5, 0) gives forward and backward
    residuals of exactly 1.5 px, an error of exactly 3.0 (= threshold_px)."""
    t = np.array([[1.0, 0, 96.0], [0, 1.0, -8.0], [0, 0, 1.0]])
    src = np.array([[10.0, 20.0], [100.25, 7.5], [1023.0, 511.0], [3.0, 4.0]])
    dst = src + np.array([96.0, -8.0]) + np.array([1.5, 0.0])
    return t, src, dst


def test_ste_orc_matches_reference(orc, ref):
    for seed in range(3):
        src, dst = ste_cases(seed)
        corr = AbiWrapper.corr_array(src, dst, np.ones(len(src), np.float32))
        a = orc.symmetric_transfer_errors(H, inverse(H), corr)
        b = ref.symmetric_transfer_errors(H, inverse(H), corr)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    t, src, dst = translation_cases()
    corr = AbiWrapper.corr_array(src, dst, np.ones(len(src), np.float32))
    e = ref.symmetric_transfer_errors(t, inverse(t), corr)
    assert np.all(e == 3.0)


@pytest.mark.gpu
def test_ste_bit_exact_on_device(lp, ref):
    for seed in range(4):
        src, dst = ste_cases(seed, n=200000)
        corr = AbiWrapper.corr_array(src, dst, np.ones(len(src), np.float32))
        hi = inverse(H)
        a = lp.symmetric_transfer_errors(H, hi, corr)
        b = ref.symmetric_transfer_errors(H, hi, corr)
        diff = np.nonzero(a.view(np.uint64) != b.view(np.uint64))[0]
        assert diff.size == 0, (seed, diff[:5], a[diff[:5]], b[diff[:5]])
        # the threshold decision the estimator takes from these errors
        assert np.array_equal(a <= 3.0, b <= 3.0)
    t, src, dst = translation_cases()
    corr = AbiWrapper.corr_array(src, dst, np.ones(len(src), np.float32))
    e = lp.symmetric_transfer_errors(t, inverse(t), corr)
    assert np.all(e == 3.0)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_prosac_near_threshold(lp, ref, seed):
    """Inlier residuals drawn so that most errors lie within a few tenths of a
    pixel of the 3 px threshold: the mask, count, model and iteration count
    must equal the reference's."""
    rng = np.random.default_rng(100 + seed)
    n = 400
    src = rng.uniform(0, 1920, size=(n, 2))
    p = np.c_[src, np.ones(n)] @ H.T
    dst = p[:, :2] / p[:, 2:3]
    k = int(0.8 * n)
    ang = rng.uniform(0, 2 * np.pi, k)
    r = rng.uniform(1.35, 1.65, k)
    dst[:k] += np.c_[r * np.cos(ang), r * np.sin(ang)]
    dst[k:] = rng.uniform(0, 1920, size=(n - k, 2))
    q = np.linspace(1.0, 0.5, n).astype(np.float32)
    corr = AbiWrapper.corr_array(src, dst, q)
    cfg = ref.default_params().prosac
    cfg.seed = seed
    a = lp.prosac_homography(corr, cfg)
    b = ref.prosac_homography(corr, cfg)
    assert a["iterations"] == b["iterations"]
    assert a["inlier_count"] == b["inlier_count"]
    assert np.array_equal(a["mask"], b["mask"])
    assert np.array_equal(a["model"], b["model"])


def test_glibc_hypot_restatement_matches_libm(tmp_path):
    """oracle/hypot_check.c: the algorithm homography.cu's glibc_hypot runs,
    compiled for the host without FMA contraction, against libm's hypot."""
    import os
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "hypot_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(root, "oracle", "hypot_check.c"),
                    "-lm"], check=True)
    r = subprocess.run([exe, "2000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
