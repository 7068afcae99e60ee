"""numpy-level wrappers over the C-ABI (include/lorbpano_b200.h).

AbiWrapper maps the reference's function names (lorb.hpp, matchlsh.hpp,
homography.hpp, compose.hpp, imgops.hpp) onto the lp_*/ref_*/orc_* entry
points, so the product (paper_1810_03988_b200.lib.Lorb) and the test oracles
expose the same calls and tests read like the reference's own.
Keypoints travel as int32 (n,4) rows (x, y, response-bits, region_id) and
descriptors as uint64 (n, 2W) rows (gt words then lt words).
"""
import ctypes as C

import numpy as np

from . import abi


def _ptr(a):
    """numpy array -> void*; torch tensors (device or host) pass their data_ptr."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


class AbiWrapper:

    lib = None
    prefix = ""
    ctx_args = ()

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _call(self, name, *args):
        st = self._fn(name)(*self.ctx_args, *args)
        if st != 0:
            raise abi.LorbError(st, self._fn("last_error")().decode())

    # ---- params ----
    def default_params(self):
        p = abi.Params()
        self._fn("params_default")(C.byref(p))
        return p

    # ---- synth (reference only) ----
    def texture(self, w, h, seed, sigma=1.5):
        out = np.zeros((h, w), np.uint8)
        self._call("synth_texture", w, h, seed, sigma, _ptr(out))
        return out

    def planted_pair(self, w, h, overlap=0.25, seed=42):
        l = np.zeros((h, w), np.uint8)
        r = np.zeros((h, w), np.uint8)
        th = np.zeros(9, np.float64)
        self._call("synth_planted_pair", w, h, overlap, seed, _ptr(l), _ptr(r), _ptr(th))
        return l, r, th

    def sequence_frame(self, w, h, frame, overlap=0.25, seed=42):
        l = np.zeros((h, w), np.uint8)
        r = np.zeros((h, w), np.uint8)
        self._call("synth_sequence_frame", w, h, overlap, seed, frame, _ptr(l), _ptr(r))
        return l, r

    def rotate(self, img, degrees):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.zeros_like(img)
        self._call("synth_rotate", _ptr(img), img.shape[1], img.shape[0], degrees, _ptr(out))
        return out

    # ---- lorb ----
    def partition_regions(self, dims, overlap=0.25, patch_half=15):
        d = np.ascontiguousarray(np.array(dims, np.int32).reshape(-1))
        out = (abi.Region * 64)()
        n = C.c_int()
        self._call("partition_regions", _ptr(d), len(dims), overlap, patch_half, out, 64,
                   C.byref(n))
        return [tuple(getattr(out[i], f) for f in ("x0", "y0", "x1", "y1", "camera_id"))
                for i in range(n.value)]

    def brief_pattern(self, n_d=256, patch_half=15, seed=42):
        out = np.zeros((n_d, 4), np.int32)
        self._call("brief_pattern", n_d, patch_half, seed, _ptr(out))
        return out

    def fast_corners(self, img, region, threshold=20, arc=9):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        ch = 1 if img.ndim == 2 else img.shape[2]
        cap = w * h
        xy = np.zeros((cap, 2), np.int32)
        n = C.c_int()
        self._call("fast_corners", _ptr(img), w, h, ch, abi.Region(*region), threshold, arc,
                   _ptr(xy), cap, C.byref(n))
        return xy[:n.value].copy()

    def harris_response(self, img, xy, alpha=0.04, sigma=1.0):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        ch = 1 if img.ndim == 2 else img.shape[2]
        xy = np.ascontiguousarray(xy, np.int32).reshape(-1, 2)
        out = np.zeros(len(xy), np.float32)
        self._call("harris_response", _ptr(img), w, h, ch, _ptr(xy), len(xy), alpha, sigma,
                   _ptr(out))
        return out

    @staticmethod
    def kp_array(kps):
        """list of (x, y, response, region_id) or structured array -> int32 (n,4) view."""
        a = np.zeros((len(kps), 4), np.int32)
        if len(kps):
            kps = np.asarray(kps)
            a[:, 0] = kps[:, 0]
            a[:, 1] = kps[:, 1]
            a[:, 2] = np.asarray(kps[:, 2], np.float32).view(np.int32)
            a[:, 3] = kps[:, 3]
        return a

    def nms(self, kp, radius=1):
        kp = np.ascontiguousarray(kp, np.int32).reshape(-1, 4)
        out = np.zeros_like(kp)
        n = C.c_int()
        self._call("nms", _ptr(kp), len(kp), radius, _ptr(out), C.byref(n))
        return out[:n.value].copy()

    def select_top_n(self, kp, top_n):
        kp = np.ascontiguousarray(kp, np.int32).reshape(-1, 4)
        out = np.zeros_like(kp)
        n = C.c_int()
        self._call("select_top_n", _ptr(kp), len(kp), top_n, _ptr(out), C.byref(n))
        return out[:n.value].copy()

    def gaussian_kernel(self, sigma):
        out = np.zeros(256, np.float32)
        n = C.c_int()
        self._call("gaussian_kernel", sigma, _ptr(out), C.byref(n))
        return out[:n.value].copy()

    def gaussian_blur(self, img, sigma):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape[:2]
        ch = 1 if img.ndim == 2 else img.shape[2]
        out = np.zeros_like(img)
        self._call("gaussian_blur", _ptr(img), w, h, ch, sigma, _ptr(out))
        return out

    def brief_descriptors(self, smoothed, kp, pairs, patch_half=15):
        sm = np.ascontiguousarray(smoothed, np.float32)
        kp = np.ascontiguousarray(kp, np.int32).reshape(-1, 4)
        pairs = np.ascontiguousarray(pairs, np.int32)
        n_d = len(pairs)
        W = (n_d + 63) // 64
        out = np.zeros((len(kp), 2 * W), np.uint64)
        self._call("brief_descriptors", _ptr(sm), sm.shape[1], sm.shape[0], _ptr(kp), len(kp),
                   _ptr(pairs), n_d, patch_half, _ptr(out))
        return out

    def extract_features(self, img, regions, cfg, pairs):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape[:2]
        ch = 1 if img.ndim == 2 else img.shape[2]
        regs = np.ascontiguousarray(np.array(regions, np.int32).reshape(-1, 5))
        cap = max(1, len(regions) * cfg.top_n)
        W = (cfg.n_d + 63) // 64
        kp = np.zeros((cap, 4), np.int32)
        desc = np.zeros((cap, 2 * W), np.uint64)
        n = C.c_int()
        pairs = np.ascontiguousarray(pairs, np.int32)
        self._call("extract_features", _ptr(img), w, h, ch, _ptr(regs), len(regs), C.byref(cfg),
                   _ptr(pairs), _ptr(kp), _ptr(desc), cap, C.byref(n))
        return kp[:n.value].copy(), desc[:n.value].copy()

    # ---- matching ----
    def descriptor_distances(self, a, b, n_d):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        out = np.zeros(len(a), np.int32)
        self._call("descriptor_distances", _ptr(a), _ptr(b), len(a), n_d, _ptr(out))
        return out

    def lsh_bit_positions(self, n_d, tables, bits, seed):
        out = np.zeros((tables, bits), np.int32)
        self._call("lsh_bit_positions", n_d, tables, bits, seed, _ptr(out))
        return out

    def probe_sequence(self, k, t):
        out = np.zeros(t, np.uint64)
        self._call("probe_sequence", k, t, _ptr(out))
        return out

    def match_features(self, a, b, n_d, cfg):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        cap = max(1, len(a))
        out = np.zeros((cap, 4), np.int32)
        n = C.c_int()
        self._call("match_features", _ptr(a), len(a), _ptr(b), len(b), n_d, C.byref(cfg),
                   _ptr(out), cap, C.byref(n))
        return out[:n.value].copy()

    def lsh_query(self, train, queries, n_d, cfg, query_id0=0):
        """query (matchlsh.hpp:132-159) of every query against build_index(train):
        (offsets (nq + 1), hits (total, 4) as lp_match rows)."""
        train = np.ascontiguousarray(train, np.uint64)
        queries = np.ascontiguousarray(queries, np.uint64)
        nq = len(queries)
        offsets = np.zeros(nq + 1, np.int64)
        total = C.c_longlong()
        cap = max(1, nq * 8)
        while True:
            out = np.zeros((cap, 4), np.int32)
            self._call("lsh_query", _ptr(train), len(train), _ptr(queries), nq, n_d, C.byref(cfg), query_id0,
                       _ptr(offsets), _ptr(out), C.c_longlong(cap), C.byref(total))
            if total.value <= cap:
                return offsets, out[:total.value].copy()
            cap = total.value

    # ---- homography ----
    @staticmethod
    def corr_array(src, dst, quality):
        n = len(src)
        a = np.zeros(n, dtype=[("sx", "f8"), ("sy", "f8"), ("dx", "f8"), ("dy", "f8"),
                               ("q", "f4"), ("pad", "i4")])
        a["sx"], a["sy"] = np.asarray(src, float)[:, 0], np.asarray(src, float)[:, 1]
        a["dx"], a["dy"] = np.asarray(dst, float)[:, 0], np.asarray(dst, float)[:, 1]
        a["q"] = quality
        return a

    def dlt_homography(self, corr):
        h = abi.Homography()
        self._call("dlt_homography", _ptr(corr), len(corr), C.byref(h))
        return np.array(h.h[:], np.float64).reshape(3, 3)

    def symmetric_transfer_errors(self, h, h_inv, corr):
        """symmetric_transfer_error (homography.hpp:147-152) of every pair."""
        n = len(corr)
        out = np.zeros(max(n, 1), np.float64)
        a, b = abi.Homography(), abi.Homography()
        a.h[:] = [float(v) for v in np.asarray(h, np.float64).ravel()]
        b.h[:] = [float(v) for v in np.asarray(h_inv, np.float64).ravel()]
        self._call("symmetric_transfer_errors", C.byref(a), C.byref(b), _ptr(corr), n, _ptr(out))
        return out[:n]

    def prosac_homography(self, corr, cfg, trace=False):
        n = len(corr)
        h = abi.Homography()
        mask = np.zeros(max(n, 1), np.uint8)
        cnt, it = C.c_int(), C.c_int()
        tp = np.zeros(max(cfg.max_iter, 1), np.int32) if trace else None
        ts = np.zeros((max(cfg.max_iter, 1), 4), np.int32) if trace else None
        self._call("prosac_homography", _ptr(corr), n, C.byref(cfg), C.byref(h), _ptr(mask),
                   C.byref(cnt), C.byref(it), _ptr(tp), _ptr(ts))
        res = dict(model=np.array(h.h[:]).reshape(3, 3), mask=mask[:n].astype(bool),
                   inlier_count=cnt.value, iterations=it.value)
        if trace:
            res["pool"] = tp[:it.value].copy()
            res["samples"] = ts[:it.value].copy()
        return res

    # ---- compose ----
    def compute_canvas(self, dims, homs):
        d = np.ascontiguousarray(np.array(dims, np.int32).reshape(-1))
        hs = np.ascontiguousarray(np.array(homs, np.float64).reshape(-1, 9))
        cv = abi.Canvas()
        off = np.zeros((len(dims), 2), np.int32)
        self._call("compute_canvas", _ptr(d), _ptr(hs), len(dims), C.byref(cv), _ptr(off))
        return (cv.width, cv.height, cv.origin_x, cv.origin_y), off

    def warp_image(self, img, hom, canvas):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape[:2]
        ch = 1 if img.ndim == 2 else img.shape[2]
        H = abi.Homography()
        H.h[:] = [float(v) for v in np.asarray(hom, float).reshape(-1)]
        cv = abi.Canvas(*canvas)
        shape = (cv.height, cv.width) if ch == 1 else (cv.height, cv.width, ch)
        out = np.zeros(shape, np.float32)
        cov = np.zeros((cv.height, cv.width), np.float32)
        self._call("warp_image", _ptr(img), w, h, ch, C.byref(H), C.byref(cv), _ptr(out),
                   _ptr(cov))
        return out, cov

    def linear_seam_mask(self, covs):
        covs = np.ascontiguousarray(covs, np.float32)
        n, h, w = covs.shape
        out = np.zeros_like(covs)
        self._call("linear_seam_mask", _ptr(covs), n, w, h, _ptr(out))
        return out

    def downsample(self, img):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape[:2]
        out = np.zeros((h // 2, w // 2), np.float32)
        self._call("downsample", _ptr(img), w, h, 1, _ptr(out))
        return out

    def upsample(self, img, tw, th):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape[:2]
        out = np.zeros((th, tw), np.float32)
        self._call("upsample", _ptr(img), w, h, 1, tw, th, _ptr(out))
        return out

    @staticmethod
    def level_dims(w, h, levels):
        dims = []
        for _ in range(levels):
            dims.append((w, h))
            w, h = w // 2, h // 2
        return dims

    def _unpack(self, flat, w, h, levels):
        out, off = [], 0
        for lw, lh in self.level_dims(w, h, levels):
            out.append(flat[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return out

    def gaussian_pyramid(self, img, levels):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape
        flat = np.zeros(sum(a * b for a, b in self.level_dims(w, h, levels)), np.float32)
        self._call("gaussian_pyramid", _ptr(img), w, h, 1, levels, _ptr(flat))
        return self._unpack(flat, w, h, levels)

    def build_laplacian(self, img, levels):
        img = np.ascontiguousarray(img, np.float32)
        h, w = img.shape
        flat = np.zeros(sum(a * b for a, b in self.level_dims(w, h, levels)), np.float32)
        self._call("build_laplacian", _ptr(img), w, h, 1, levels, _ptr(flat))
        return self._unpack(flat, w, h, levels)

    def collapse_laplacian(self, levels_list):
        flat = np.ascontiguousarray(np.concatenate([l.reshape(-1) for l in levels_list]),
                                    np.float32)
        h, w = levels_list[0].shape
        out = np.zeros((h, w), np.float32)
        self._call("collapse_laplacian", _ptr(flat), w, h, 1, len(levels_list), _ptr(out))
        return out

    def multiband_blend(self, images, masks, levels):
        images = np.ascontiguousarray(images, np.float32)
        masks = np.ascontiguousarray(masks, np.float32)
        n, h, w = images.shape
        out = np.zeros((h, w), np.uint8)
        self._call("multiband_blend", _ptr(images), _ptr(masks), n, w, h, 1, levels, _ptr(out))
        return out

    # ---- whole frame ----
    @staticmethod
    def cameras(specs):
        """[(pre_transform 3x3 or None, crop (x0, y0, x1, y1) or None), ...] -> Camera array."""
        arr = (abi.Camera * len(specs))()
        for c, (hom, crop) in enumerate(specs):
            h = np.eye(3) if hom is None else np.asarray(hom, np.float64).reshape(3, 3)
            arr[c].pre_transform.h[:] = list(h.ravel())
            arr[c].has_crop = 0 if crop is None else 1
            if crop is not None:
                arr[c].crop = abi.Region(*[int(v) for v in crop], c)
        return arr

    def rectify_crop(self, images, specs):
        """stage_rectify_crop (pipeline.hpp:391-417): list of u8 images."""
        ncams = len(images)
        h, w = images[0].shape
        imgs = [np.ascontiguousarray(i, np.uint8) for i in images]
        outs = [np.zeros(w * h, np.uint8) for _ in images]
        ow = np.zeros(ncams, np.int32)
        oh = np.zeros(ncams, np.int32)
        self._call("rectify_crop", ncams, w, h, self.cameras(specs),
                   (C.c_void_p * ncams)(*[i.ctypes.data for i in imgs]),
                   (C.c_void_p * ncams)(*[o.ctypes.data for o in outs]),
                   ow.ctypes.data_as(abi.c_intp), oh.ctypes.data_as(abi.c_intp))
        return [outs[c][:ow[c] * oh[c]].reshape(oh[c], ow[c]).copy() for c in range(ncams)]

    def stitch_frame(self, images, params, frame_index=0, pano_cap=None, cameras=None):
        ncams = len(images)
        h, w = images[0].shape
        imgs = [np.ascontiguousarray(i, np.uint8) for i in images]
        ptrs = (C.c_void_p * ncams)(*[i.ctypes.data for i in imgs])
        cap_kp = 2 * params.extraction.top_n
        W = (params.extraction.n_d + 63) // 64
        pano_cap = pano_cap or (ncams * w * 2 * h)
        pano = np.zeros(pano_cap, np.uint8)
        homs = (abi.Homography * ncams)()
        kpc = np.zeros(ncams, np.int32)
        kps = np.zeros((ncams, cap_kp, 4), np.int32)
        desc = np.zeros((ncams, cap_kp, 2 * W), np.uint64)
        mc = np.zeros(max(ncams - 1, 1), np.int32)
        cap_m = cap_kp
        mt = np.zeros((max(ncams - 1, 1), cap_m, 4), np.int32)
        fo = abi.FrameOut()
        fo.panorama = pano.ctypes.data_as(abi.c_u8p)
        fo.pano_cap = pano_cap
        fo.homographies = homs
        fo.kp_counts = kpc.ctypes.data_as(abi.c_intp)
        fo.keypoints = kps.ctypes.data_as(C.POINTER(abi.Keypoint))
        fo.descriptors = desc.ctypes.data_as(abi.c_u64p)
        fo.cap_kp = cap_kp
        fo.match_counts = mc.ctypes.data_as(abi.c_intp)
        fo.matches = mt.ctypes.data_as(C.POINTER(abi.Match))
        fo.cap_matches = cap_m
        if cameras is None:
            self._call("stitch_frame", ncams, w, h, C.byref(params), ptrs, frame_index, C.byref(fo))
        else:  # RigLayout (reference only)
            self._call("stitch_frame_layout", ncams, w, h, self.cameras(cameras), C.byref(params), ptrs,
                       frame_index, C.byref(fo))
        cv = fo.canvas
        return dict(
            canvas=(cv.width, cv.height, cv.origin_x, cv.origin_y),
            panorama=pano[:cv.width * cv.height].reshape(cv.height, cv.width).copy(),
            homographies=np.array([homs[i].h[:] for i in range(ncams)]).reshape(ncams, 3, 3),
            keypoints=[kps[c, :kpc[c]].copy() for c in range(ncams)],
            descriptors=[desc[c, :kpc[c]].copy() for c in range(ncams)],
            matches=[mt[p, :mc[p]].copy() for p in range(ncams - 1)],
        )
