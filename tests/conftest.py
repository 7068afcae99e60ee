"""Shared fixtures. Parity tests compare the CUDA path (through the C-ABI) with
the plain-C restatement oracle (oracle/lorb_oracle.c), itself pinned to the
reference by tests/test_oracle_golden.py."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built CUDA library")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, ref_available
    if not ref_available():
        pytest.skip("reference oracle (oracle/_ref) not built here")
    return Oracle("ref")


@pytest.fixture(scope="session")
def lp():
    from paper_1810_03988_b200 import Lorb
    return Lorb(0)


@pytest.fixture(scope="session")
def params(orc):
    p = orc.default_params()
    p.seed = 42
    p.matching.seed = 42  # config.hpp:212 sets matching.seed = seed on the CLI path
    return p


def rand_image(w, h, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)


def chain_cameras(o, ncams, w, h, overlap=0.25, seed=42):
    """N-camera horizontal chain cut from one wide texture (cli.hpp:311-322)."""
    shift = int(np.floor(w * (1.0 - overlap) + 0.5))
    wide = o.texture(w + shift * (ncams - 1), h, seed)
    cams = [np.ascontiguousarray(wide[:, c * shift:c * shift + w]) for c in range(ncams)]
    return cams, wide, shift
