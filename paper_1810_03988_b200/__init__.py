"""paper_1810_03988_b200 — B200-native per-frame panorama stitching hot path of
arXiv 1810.03988 (reference `lorbpano`): L-ORB extraction, multi-probe LSH
matching, PROSAC homography, warp + multi-band blend, as sm_100a kernels behind
the C-ABI in include/lorbpano_b200.h.

    from paper_1810_03988_b200 import Lorb, Rig
    lp = Lorb()                        # one context on cuda:0
    rig = Rig(lp, ncams, w, h, lp.default_params())
    out = rig.stitch([cam0, cam1])     # panorama + homographies
"""
from .abi import LorbError  # noqa: F401
from .lib import Lorb, Rig, build, frame_out, kernel_launches, load  # noqa: F401
from . import abi  # noqa: F401
