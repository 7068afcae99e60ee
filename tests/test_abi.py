"""CPU-side checks of the C-ABI boundary: the in-tree CUDA library loads,
exports every entry point include/lorbpano_b200.h declares, fills the
reference defaults, and fails loudly (NoDevice) instead of falling back to
the CPU when no GPU is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lorbpano_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1810_03988_b200 import lib as L
    return L.load()


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("lp_fast_corners", "lp_harris_response", "lp_nms", "lp_select_top_n",
              "lp_extract_features", "lp_match_features", "lp_prosac_homography",
              "lp_warp_image", "lp_multiband_blend", "lp_rig_create", "lp_rig_stitch"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_defaults_match_reference(lib, orc):
    from paper_1810_03988_b200 import abi
    a, b = abi.Params(), abi.Params()
    lib.lp_params_default(C.byref(a))
    b = orc.default_params()
    assert bytes(a) == bytes(b)


def test_defaults_match_reference_itself(lib, ref):
    from paper_1810_03988_b200 import abi
    a = abi.Params()
    lib.lp_params_default(C.byref(a))
    assert bytes(a) == bytes(ref.default_params())


def test_no_silent_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1810_03988_b200 import Lorb, LorbError
    with pytest.raises(LorbError) as e:
        Lorb(0)
    assert e.value.name == "NoDevice"


def test_synth_texture_is_the_references():
    """lp_synth_texture (the bench's input generator) equals the reference's
    synth::texture byte for byte (synth.hpp:17-34)."""
    import numpy as np
    from oracle import Oracle, ref_available
    from paper_1810_03988_b200.lib import synth_texture
    if not ref_available():
        pytest.skip("reference oracle (oracle/_ref) not built here")
    ref = Oracle("ref")
    for w, h, seed, sigma in ((160, 120, 7, 1.5), (641, 479, 42, 1.5), (333, 251, 9, 2.0)):
        assert np.array_equal(synth_texture(w, h, seed, sigma), ref.texture(w, h, seed, sigma))
