"""Python host side of the B200 stitching path: loads the in-tree CUDA library
(_lib/liblorbpano_b200.so) and exposes the reference's function names through
the C-ABI. There is no CPU fallback: if the library or a GPU is missing, the
calls fail loudly (LorbError NoDevice / ImportError)."""
import ctypes as C
import os
import subprocess
import threading

import numpy as np

from . import abi
from .api import AbiWrapper, _ptr

HERE = os.path.dirname(os.path.abspath(__file__))
# LPB_LIB selects an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("LPB_LIB") or os.path.join(HERE, "_lib", "liblorbpano_b200.so")
CSRC = os.path.join(HERE, "csrc")

_lock = threading.Lock()
_lib = None


def build(jobs=8):
    """Compile csrc/*.cu for sm_100a into _lib/liblorbpano_b200.so (make, in-tree)."""
    r = subprocess.run(["make", "-s", f"-j{jobs}", "-f", os.path.join(CSRC, "Makefile")],
                       cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("CUDA build failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])
    return LIB_PATH


def load():
    """The product library (built in-tree if absent). Raises if it cannot be had."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            build()
        lib = C.CDLL(LIB_PATH)
        abi.bind(lib, "lp_", with_ctx=True)
        P = C.c_void_p
        lib.lp_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
        lib.lp_ctx_create.restype = C.c_int
        lib.lp_ctx_destroy.argtypes = [P]
        lib.lp_ctx_destroy.restype = None
        lib.lp_ctx_set_stream.argtypes = [P, P]
        lib.lp_ctx_set_stream.restype = C.c_int
        lib.lp_kernel_launches.argtypes = []
        lib.lp_kernel_launches.restype = C.c_uint64
        lib.lp_params_default.argtypes = [C.POINTER(abi.Params)]
        lib.lp_params_default.restype = None
        lib.lp_rig_create.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(abi.Params), C.POINTER(P)]
        lib.lp_rig_create.restype = C.c_int
        lib.lp_rig_create_layout.argtypes = [P, C.c_int, C.c_int, C.c_int, P, C.POINTER(abi.Params),
                                             C.POINTER(P)]
        lib.lp_rig_create_layout.restype = C.c_int
        lib.lp_brief_pattern.argtypes = [C.c_int, C.c_int, C.c_uint64, P]
        lib.lp_brief_pattern.restype = C.c_int
        lib.lp_load_pnm.argtypes = [C.c_char_p, P, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int)]
        lib.lp_load_pnm.restype = C.c_int
        lib.lp_save_pnm.argtypes = [C.c_char_p, P, C.c_int, C.c_int, C.c_int]
        lib.lp_save_pnm.restype = C.c_int
        lib.lp_gray_to_rgb.argtypes = [P, P, C.c_size_t, P]
        lib.lp_gray_to_rgb.restype = C.c_int
        lib.lp_rig_set_egress.argtypes = [P, C.c_int]
        lib.lp_rig_set_egress.restype = C.c_int
        lib.lp_rig_destroy.argtypes = [P]
        lib.lp_rig_destroy.restype = None
        lib.lp_host_alloc.argtypes = [C.c_size_t]
        lib.lp_host_alloc.restype = P
        lib.lp_host_alloc_wc.argtypes = [C.c_size_t]
        lib.lp_host_alloc_wc.restype = P
        lib.lp_host_free.argtypes = [P]
        lib.lp_host_free.restype = None
        lib.lp_synth_texture.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_float, P]
        lib.lp_synth_texture.restype = C.c_int
        lib.lp_rig_stitch.argtypes = [P, P, C.c_uint64, C.POINTER(abi.FrameOut)]
        lib.lp_rig_stitch.restype = C.c_int
        lib.lp_rig_panorama_capacity.argtypes = [P]
        lib.lp_rig_panorama_capacity.restype = C.c_size_t
        lib.lp_rig_stream.argtypes = [P]
        lib.lp_rig_stream.restype = P
        lib.lp_rig_submit.argtypes = [P, P, C.c_uint64, P, C.c_size_t, C.POINTER(C.c_uint64)]
        lib.lp_rig_submit.restype = C.c_int
        lib.lp_rig_wait.argtypes = [P, C.c_uint64, C.POINTER(abi.Canvas)]
        lib.lp_rig_wait.restype = C.c_int
        lib.lp_rig_submit_frame.argtypes = [P, P, C.c_uint64, C.POINTER(abi.FrameOut), C.POINTER(C.c_uint64)]
        lib.lp_rig_submit_frame.restype = C.c_int
        lib.lp_rig_wait_frame.argtypes = [P, C.c_uint64, C.POINTER(abi.FrameOut)]
        lib.lp_rig_wait_frame.restype = C.c_int
        lib.lp_rig_set_graphs.argtypes = [P, C.c_int]
        lib.lp_rig_set_graphs.restype = C.c_int
        lib.lp_rig_set_streams.argtypes = [P, C.c_int]
        lib.lp_rig_set_streams.restype = C.c_int
        lib.lp_rig_inject_fault.argtypes = [P, C.c_uint64, C.c_int]
        lib.lp_rig_inject_fault.restype = C.c_int
        lib.lp_rig_algorithmic_bytes.argtypes = [P, C.c_char_p]
        lib.lp_rig_algorithmic_bytes.restype = C.c_double
        lib.lp_rig_algorithmic_work.argtypes = [P, C.c_char_p, C.c_longlong, C.POINTER(C.c_double)]
        lib.lp_rig_algorithmic_work.restype = C.c_int
        lib.lp_rig_work_reset.argtypes = [P]
        lib.lp_rig_work_reset.restype = C.c_int
        lib.lp_rig_reset.argtypes = [P]
        lib.lp_rig_reset.restype = C.c_int
        lib.lp_rig_copy_panorama.argtypes = [P, C.c_uint64, P, C.c_size_t]
        lib.lp_rig_copy_panorama.restype = C.c_int
        lib.lp_profile_enable.argtypes = [C.c_int]
        lib.lp_profile_enable.restype = None
        lib.lp_profile_reset.argtypes = []
        lib.lp_profile_reset.restype = None
        _lib = lib
        return lib


def kernel_launches():
    return int(load().lp_kernel_launches())


def frame_out(pano_ptr, pano_cap):
    """A FrameOut that only receives the panorama (host or device address):
    with a device address lp_rig_stitch returns without synchronising."""
    fo = abi.FrameOut()
    fo.panorama = C.cast(C.c_void_p(pano_ptr), abi.c_u8p)
    fo.pano_cap = pano_cap
    return fo


def _check(lib, st):
    if st != 0:
        raise abi.LorbError(st, lib.lp_last_error().decode())


class Lorb(AbiWrapper):
    """The reference's L1 API (lorb/matchlsh/homography/compose/imgops) on the GPU."""

    def __init__(self, device=0):
        self.lib = load()
        self.prefix = "lp_"
        ctx = C.c_void_p()
        _check(self.lib, self.lib.lp_ctx_create(device, C.byref(ctx)))
        self.ctx = ctx
        self.ctx_args = (ctx,)

    def close(self):
        if self.ctx:
            self.lib.lp_ctx_destroy(self.ctx)
            self.ctx = None
            self.ctx_args = ()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def default_params(self):
        p = abi.Params()
        self.lib.lp_params_default(C.byref(p))
        return p

    def brief_pattern(self, n_d=256, patch_half=15, seed=42):
        """brief_pattern (lorb.hpp:303-330), host side of the product library."""
        out = np.zeros((n_d, 4), np.int32)
        _check(self.lib, self.lib.lp_brief_pattern(n_d, patch_half, seed, out.ctypes.data))
        return out

    def gray_to_rgb(self, gray):
        """The PPM sink's triplication (cli.hpp:138-145) on the device."""
        g = np.ascontiguousarray(gray, np.uint8)
        out = np.empty(g.shape + (3,), np.uint8)
        _check(self.lib, self.lib.lp_gray_to_rgb(self.ctx, g.ctypes.data, g.size, out.ctypes.data))
        return out

    def stitch_frame(self, images, params, frame_index=0, pano_cap=None, cameras=None):
        """One frame through a fresh engine (the oracles' stitch_frame);
        `cameras` = RigLayout specs as for rectify_crop."""
        h, w = images[0].shape[:2]
        rig = Rig(self, len(images), w, h, params, cameras=cameras)
        try:
            return rig.stitch(images, frame_index, pano_cap=pano_cap, details=True)
        finally:
            rig.close()


class Rig:
    """StitchEngine for a chain of identical cameras (pipeline.hpp:341-721) on one GPU."""

    def __init__(self, lorb, ncams, w, h, params, cameras=None):
        self.lorb = lorb
        self.lib = lorb.lib
        self.ncams, self.w, self.h = ncams, w, h
        self.params = params
        r = C.c_void_p()
        if cameras is None:
            _check(self.lib, self.lib.lp_rig_create(lorb.ctx, ncams, w, h, C.byref(params), C.byref(r)))
        else:  # RigLayout: stage_rectify_crop on ingest
            cams = AbiWrapper.cameras(cameras)
            _check(self.lib, self.lib.lp_rig_create_layout(lorb.ctx, ncams, w, h, cams, C.byref(params),
                                                           C.byref(r)))
        self.rig = r

    def reset(self):
        """A fresh HomographyCache on this rig's device resources (lp_rig_reset)."""
        _check(self.lib, self.lib.lp_rig_reset(self.rig))

    def close(self):
        if self.rig:
            self.lib.lp_rig_destroy(self.rig)
            self.rig = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_graphs(self, on=True):
        """Replay the compositor chain as a CUDA graph per frame slot (default on)."""
        _check(self.lib, self.lib.lp_rig_set_graphs(self.rig, 1 if on else 0))

    def inject_fault(self, frame_index, code):
        """The frame submitted with `frame_index` fails with device status
        `code` (lp_rig_inject_fault); only that frame's wait() raises."""
        _check(self.lib, self.lib.lp_rig_inject_fault(self.rig, frame_index, code))

    def set_egress_rgb(self, on=True):
        """Panoramas leave the device as 3-channel RGB (the PPM sink's format)."""
        _check(self.lib, self.lib.lp_rig_set_egress(self.rig, 1 if on else 0))

    @property
    def stream(self):
        return self.lib.lp_rig_stream(self.rig)

    def panorama_capacity(self):
        return int(self.lib.lp_rig_panorama_capacity(self.rig))

    def submit(self, image_ptrs, frame_index, pano_ptr=None, pano_cap=0):
        """Asynchronous frame (lp_rig_submit): returns a ticket for wait()."""
        arr = (C.c_void_p * self.ncams)(*image_ptrs)
        t = C.c_uint64()
        _check(self.lib, self.lib.lp_rig_submit(self.rig, arr, frame_index, pano_ptr, pano_cap, C.byref(t)))
        return t.value

    def wait(self, ticket):
        cv = abi.Canvas()
        _check(self.lib, self.lib.lp_rig_wait(self.rig, ticket, C.byref(cv)))
        return (cv.width, cv.height, cv.origin_x, cv.origin_y)

    def stitch_raw(self, image_ptrs, frame_index, fo):
        """Zero-copy call: image_ptrs = list of addresses (host or device), fo a FrameOut."""
        arr = (C.c_void_p * self.ncams)(*image_ptrs)
        _check(self.lib, self.lib.lp_rig_stitch(self.rig, arr, frame_index, C.byref(fo)))

    def _frame_out(self, images, pano_cap, details):
        """Host buffers + FrameOut for one frame (keeps the arrays alive)."""
        ptrs = []
        keep = []
        for im in images:
            if hasattr(im, "data_ptr"):
                ptrs.append(im.data_ptr())
            else:
                a = np.ascontiguousarray(im, np.uint8)
                keep.append(a)
                ptrs.append(a.ctypes.data)
        p = self.params
        ncams = self.ncams
        pano_cap = pano_cap or self.panorama_capacity()
        st = dict(ptrs=ptrs, keep=keep, details=details)
        st["pano"] = np.zeros(pano_cap, np.uint8)
        st["homs"] = (abi.Homography * ncams)()
        fo = abi.FrameOut()
        fo.panorama = st["pano"].ctypes.data_as(abi.c_u8p)
        fo.pano_cap = pano_cap
        fo.homographies = st["homs"]
        if details:
            cap_kp = 2 * p.extraction.top_n
            W = (p.extraction.n_d + 63) // 64
            st["kpc"] = np.zeros(ncams, np.int32)
            st["kps"] = np.zeros((ncams, cap_kp, 4), np.int32)
            st["desc"] = np.zeros((ncams, cap_kp, 2 * W), np.uint64)
            st["mc"] = np.zeros(max(ncams - 1, 1), np.int32)
            st["mt"] = np.zeros((max(ncams - 1, 1), cap_kp, 4), np.int32)
            fo.kp_counts = st["kpc"].ctypes.data_as(abi.c_intp)
            fo.keypoints = st["kps"].ctypes.data_as(C.POINTER(abi.Keypoint))
            fo.descriptors = st["desc"].ctypes.data_as(abi.c_u64p)
            fo.cap_kp = cap_kp
            fo.match_counts = st["mc"].ctypes.data_as(abi.c_intp)
            fo.matches = st["mt"].ctypes.data_as(C.POINTER(abi.Match))
            fo.cap_matches = cap_kp
        st["fo"] = fo
        return st

    def _result(self, st):
        fo, ncams = st["fo"], self.ncams
        cv = fo.canvas
        homs = st["homs"]
        out = dict(
            canvas=(cv.width, cv.height, cv.origin_x, cv.origin_y),
            panorama=st["pano"][:cv.width * cv.height].reshape(cv.height, cv.width).copy(),
            homographies=np.array([homs[i].h[:] for i in range(ncams)]).reshape(ncams, 3, 3),
            estimated=bool(fo.estimated),
            stage_ms=list(fo.stage_ms),
        )
        if st["details"]:
            kpc, kps, desc, mc, mt = st["kpc"], st["kps"], st["desc"], st["mc"], st["mt"]
            out.update(
                keypoints=[kps[c, :kpc[c]].copy() for c in range(ncams)],
                descriptors=[desc[c, :kpc[c]].copy() for c in range(ncams)],
                matches=[mt[q, :mc[q]].copy() for q in range(ncams - 1)],
            )
        return out

    def stitch(self, images, frame_index=0, pano_cap=None, details=False):
        st = self._frame_out(images, pano_cap, details)
        self.stitch_raw(st["ptrs"], frame_index, st["fo"])
        return self._result(st)

    def submit_frame(self, images, frame_index, details=True, pano_cap=None):
        """Frame in flight with its per-frame results (lp_rig_submit_frame);
        wait_frame(handle) returns them as stitch(details=True) does."""
        st = self._frame_out(images, pano_cap, details)
        arr = (C.c_void_p * self.ncams)(*st["ptrs"])
        t = C.c_uint64()
        _check(self.lib, self.lib.lp_rig_submit_frame(self.rig, arr, frame_index, C.byref(st["fo"]), C.byref(t)))
        st["ticket"] = t.value
        return st

    def wait_frame(self, st):
        code = self.lib.lp_rig_wait_frame(self.rig, st["ticket"], C.byref(st["fo"]))
        fo = st["fo"]
        if code == 24 and fo.canvas.width > 0 and fo.canvas.height > 0:
            # the canvas outgrew the panorama buffer: the frame is stitched,
            # its panorama waits in the rig (lp_rig_copy_panorama)
            need = fo.canvas.width * fo.canvas.height
            st["pano"] = np.zeros(need, np.uint8)
            fo.panorama = st["pano"].ctypes.data_as(abi.c_u8p)
            fo.pano_cap = need
            code = self.lib.lp_rig_copy_panorama(self.rig, st["ticket"], st["pano"].ctypes.data, need)
        _check(self.lib, code)
        return self._result(st)


def synth_texture(w, h, seed, sigma=1.5):
    """synth::texture (synth.hpp:17-34) through the C-ABI (host only)."""
    lib = load()
    out = np.empty((h, w), np.uint8)
    _check(lib, lib.lp_synth_texture(w, h, seed, sigma, out.ctypes.data))
    return out


def load_pnm(path):
    """load_pnm (image.hpp:88-126) through the C-ABI: (h, w) or (h, w, 3) uint8."""
    lib = load()
    w, h, ch = C.c_int(), C.c_int(), C.c_int()
    p = os.fsencode(path)
    _check(lib, lib.lp_load_pnm(p, None, 0, C.byref(w), C.byref(h), C.byref(ch)))
    shape = (h.value, w.value) if ch.value == 1 else (h.value, w.value, 3)
    out = np.empty(shape, np.uint8)
    _check(lib, lib.lp_load_pnm(p, out.ctypes.data, out.size, C.byref(w), C.byref(h), C.byref(ch)))
    return out


def save_pnm(path, img):
    """save_pnm (image.hpp:194-204): P5 for (h, w), P6 for (h, w, 3)."""
    lib = load()
    a = np.ascontiguousarray(img, np.uint8)
    ch = 1 if a.ndim == 2 else a.shape[2]
    _check(lib, lib.lp_save_pnm(os.fsencode(path), a.ctypes.data, a.shape[1], a.shape[0], ch))
