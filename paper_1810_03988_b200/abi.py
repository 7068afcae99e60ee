"""ctypes mirror of include/lorbpano_b200.h (the C-ABI boundary).

The same prototypes are bound for three libraries that share the signatures:
  lp_*   the CUDA product   (paper_1810_03988_b200/_lib/liblorbpano_b200.so)
  ref_*  the reference itself compiled as an oracle (oracle/_ref/liblorbref.so)
  orc_*  the C restatement oracle (oracle/_build/liborc.so)
ref_/orc_ functions take no context argument.
"""
import ctypes as C

c_u8p = C.POINTER(C.c_uint8)
c_u64p = C.POINTER(C.c_uint64)
c_intp = C.POINTER(C.c_int)
c_fp = C.POINTER(C.c_float)
c_dp = C.POINTER(C.c_double)

STATUS_NAMES = {
    0: "OK", 1: "FileNotFound", 2: "UnsupportedFormat", 3: "CorruptData", 4: "InvalidSigma",
    5: "ImageTooSmall", 6: "BadTargetDims", 7: "NoOverlap", 8: "OverlapExceedsImage",
    9: "RegionTooSmall", 10: "WindowOutOfBounds", 11: "PatchOutOfBounds", 12: "LengthMismatch",
    13: "BadParams", 14: "TooManyProbes", 15: "ParamMismatch", 16: "EmptyInput",
    17: "DegenerateConfiguration", 18: "NumericalFailure", 19: "InsufficientMatches",
    20: "NoModelFound", 21: "SingularHomography", 22: "MaskMismatch", 23: "TooManyLevels",
    24: "CapacityOverflow", 25: "NoValidHomographyYet", 26: "ParseError", 27: "ValidationError",
    28: "MissingFrames", 100: "CudaError", 101: "NoDevice", 102: "Internal",
}


class LorbError(RuntimeError):
    """Raised for a non-zero lp_status; `.name` is the lorbpano::Error subclass name."""

    def __init__(self, code, msg=""):
        self.code = code
        self.name = STATUS_NAMES.get(code, f"status{code}")
        super().__init__(f"{self.name}: {msg}")


class Region(C.Structure):
    _fields_ = [("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int), ("y1", C.c_int),
                ("camera_id", C.c_int)]


class Keypoint(C.Structure):
    _fields_ = [("x", C.c_int), ("y", C.c_int), ("response", C.c_float), ("region_id", C.c_int)]


class Pair(C.Structure):
    _fields_ = [("px", C.c_int), ("py", C.c_int), ("qx", C.c_int), ("qy", C.c_int)]


class Match(C.Structure):
    _fields_ = [("query_id", C.c_int), ("train_id", C.c_int), ("distance", C.c_int),
                ("quality", C.c_float)]


class Corr(C.Structure):
    _fields_ = [("sx", C.c_double), ("sy", C.c_double), ("dx", C.c_double), ("dy", C.c_double),
                ("quality", C.c_float), ("pad_", C.c_int)]


class Homography(C.Structure):
    _fields_ = [("h", C.c_double * 9)]


class Camera(C.Structure):
    """RigLayout::Camera (pipeline.hpp:240-247): pre_transform + optional crop."""
    _fields_ = [("pre_transform", Homography), ("has_crop", C.c_int), ("crop", Region)]


class Canvas(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("origin_x", C.c_int),
                ("origin_y", C.c_int)]


class ExtractionConfig(C.Structure):
    _fields_ = [("fast_threshold", C.c_int), ("fast_arc", C.c_int), ("harris_alpha", C.c_float),
                ("harris_threshold", C.c_float), ("harris_sigma", C.c_float), ("top_n", C.c_int),
                ("n_d", C.c_int), ("brief_blur_sigma", C.c_float), ("patch_half", C.c_int)]


class MatchConfig(C.Structure):
    _fields_ = [("tables", C.c_int), ("bits", C.c_int), ("t_probes", C.c_int),
                ("max_distance", C.c_int), ("ratio", C.c_float), ("pad_", C.c_int),
                ("seed", C.c_uint64)]


class ProsacConfig(C.Structure):
    _fields_ = [("threshold_px", C.c_double), ("max_iter", C.c_int), ("sampling", C.c_int),
                ("confidence", C.c_double), ("seed", C.c_uint64), ("t_total", C.c_double)]


class Params(C.Structure):
    _fields_ = [("extraction", ExtractionConfig), ("matching", MatchConfig),
                ("prosac", ProsacConfig), ("blend_levels", C.c_int),
                ("homography_refresh", C.c_int), ("seed", C.c_uint64),
                ("overlap_fraction", C.c_double)]


class FrameOut(C.Structure):
    _fields_ = [("panorama", c_u8p), ("pano_cap", C.c_size_t), ("canvas", Canvas),
                ("homographies", C.POINTER(Homography)), ("kp_counts", c_intp),
                ("keypoints", C.POINTER(Keypoint)), ("descriptors", c_u64p), ("cap_kp", C.c_int),
                ("match_counts", c_intp), ("matches", C.POINTER(Match)), ("cap_matches", C.c_int),
                ("estimated", C.c_int), ("stage_ms", C.c_float * 4)]


P = C.c_void_p  # generic pointer (host numpy data or device address)

# name -> argtypes after the (optional) context argument
_PROTOS = {
    "rectify_crop": [C.c_int, C.c_int, C.c_int, P, P, P, c_intp, c_intp],
    "fast_corners": [P, C.c_int, C.c_int, C.c_int, Region, C.c_int, C.c_int, P, C.c_int, c_intp],
    "harris_response": [P, C.c_int, C.c_int, C.c_int, P, C.c_int, C.c_float, C.c_float, P],
    "nms": [P, C.c_int, C.c_int, P, c_intp],
    "select_top_n": [P, C.c_int, C.c_int, P, c_intp],
    "gaussian_blur": [P, C.c_int, C.c_int, C.c_int, C.c_float, P],
    "brief_descriptors": [P, C.c_int, C.c_int, P, C.c_int, P, C.c_int, C.c_int, P],
    "extract_features": [P, C.c_int, C.c_int, C.c_int, P, C.c_int,
                         C.POINTER(ExtractionConfig), P, P, P, C.c_int, c_intp],
    "descriptor_distances": [P, P, C.c_int, C.c_int, P],
    "match_features": [P, C.c_int, P, C.c_int, C.c_int, C.POINTER(MatchConfig), P, C.c_int,
                       c_intp],
    "dlt_homography": [P, C.c_int, C.POINTER(Homography)],
    "prosac_homography": [P, C.c_int, C.POINTER(ProsacConfig), C.POINTER(Homography), P, c_intp,
                          c_intp, P, P],
    "warp_image": [P, C.c_int, C.c_int, C.c_int, C.POINTER(Homography), C.POINTER(Canvas), P, P],
    "linear_seam_mask": [P, C.c_int, C.c_int, C.c_int, P],
    "downsample": [P, C.c_int, C.c_int, C.c_int, P],
    "upsample": [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P],
    "gaussian_pyramid": [P, C.c_int, C.c_int, C.c_int, C.c_int, P],
    "build_laplacian": [P, C.c_int, C.c_int, C.c_int, C.c_int, P],
    "collapse_laplacian": [P, C.c_int, C.c_int, C.c_int, C.c_int, P],
    "multiband_blend": [P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P],
    "lsh_query": [P, C.c_int, P, C.c_int, C.c_int, C.POINTER(MatchConfig), C.c_int, P, P, C.c_longlong,
                  C.POINTER(C.c_longlong)],
}

# oracle-only helpers (ref_ and orc_)
_ORACLE_EXTRA = {
    "params_default": [C.POINTER(Params)],
    "partition_regions": [P, C.c_int, C.c_double, C.c_int, P, C.c_int, c_intp],
    "brief_pattern": [C.c_int, C.c_int, C.c_uint64, P],
    "gaussian_kernel": [C.c_float, P, c_intp],
    "lsh_bit_positions": [C.c_int, C.c_int, C.c_int, C.c_uint64, P],
    "probe_sequence": [C.c_int, C.c_int, P],
    "compute_canvas": [P, P, C.c_int, C.POINTER(Canvas), P],
    "stitch_frame": [C.c_int, C.c_int, C.c_int, C.POINTER(Params), P, C.c_uint64,
                     C.POINTER(FrameOut)],
    "synth_texture": [C.c_int, C.c_int, C.c_uint64, C.c_float, P],
    "synth_planted_pair": [C.c_int, C.c_int, C.c_double, C.c_uint64, P, P, P],
    "synth_sequence_frame": [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64, P, P],
    "synth_rotate": [P, C.c_int, C.c_int, C.c_double, P],
}

_REF_ONLY = {
    "stitch_frame_layout": [C.c_int, C.c_int, C.c_int, P, C.POINTER(Params), P, C.c_uint64,
                            C.POINTER(FrameOut)],
    "run_engine": [C.c_int, C.c_int, C.c_int, C.POINTER(Params), P, C.c_int, C.c_int, C.c_int,
                   C.c_int, c_dp, c_dp],
    "run_engines_parallel": [C.c_int, C.c_int, C.c_int, C.POINTER(Params), P, C.c_int, C.c_int,
                             c_dp],
}


def bind(lib, prefix, with_ctx):
    """Set argtypes/restype for every entry point `lib` exports under `prefix`."""
    protos = dict(_PROTOS)
    if prefix != "lp_":
        protos.update(_ORACLE_EXTRA)
    if prefix == "ref_":
        protos.update(_REF_ONLY)
    for name, args in protos.items():
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            continue
        ctx = [P] if (with_ctx and name in _PROTOS) else []
        fn.argtypes = ctx + args
        fn.restype = C.c_int
    le = getattr(lib, prefix + "last_error", None)
    if le is not None:
        le.restype = C.c_char_p
        le.argtypes = []
    return lib
