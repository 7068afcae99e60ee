"""`lorbpano` command line on the B200 path.

Mirrors tools/lorbpano_main.cpp:7-84 and cli.hpp:52-375 (CLI11 is absent, so
argparse stands in for it):

    python -m paper_1810_03988_b200 stitch  --config rig.cfg [--mode M] [--seed S]
                                            [--frames-in-flight F] [--out DIR] [--emit-timings]
    python -m paper_1810_03988_b200 extract IMAGE [--config C] [--seed S] [--out DIR]
    python -m paper_1810_03988_b200 bench   features|match|pipeline [--config C] [--out DIR]

* the config file is the reference's line-oriented `key = value` format with
  `[camera]` sections (config.hpp:84-226): same keys, same ParseError /
  ValidationError / MissingFrames behaviour, exit code 2 on configuration
  errors as the reference's main;
* frames are read with load_pnm (image.hpp:88-126, lp_load_pnm), panoramas
  leave the device already triplicated to RGB and are written as
  pano_<frame>.ppm (cli.hpp:138-147), timings.csv has the reference's columns
  (cli.hpp:74-87; per-frame rows are the rig's device stage times);
* bench suites write bench_<suite>.csv with the reference's columns
  (cli.hpp:222-358), timed on the GPU path.
Everything runs through the C-ABI (include/lorbpano_b200.h); nothing here
computes pixels on the host.
"""
import argparse
import glob
import math
import os
import sys
import time

import numpy as np

from . import abi
from .lib import Lorb, Rig, load_pnm, save_pnm

STAGES = ["ingest", "rectify_crop", "detect", "describe", "match_estimate", "warp_blend", "output"]


class ConfigError(Exception):
    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def _num(kind, value, line, key):
    try:
        if kind is int:
            if not value.lstrip("-").isdigit():
                raise ValueError
            return int(value)
        return float(value)
    except ValueError:
        raise ConfigError("ParseError", f"line {line}: bad value for {key}")


def parse_config(path, lp):
    """parse_config (config.hpp:84-226) into (params, cameras, settings)."""
    if not os.path.exists(path):
        raise ConfigError("FileNotFound", path)
    p = lp.default_params()
    cams = []
    st = dict(overlap=0.25, output_dir="out", mode="serial", frames_in_flight=4, workers_per_stage=1,
              emit_timings=False, seed=0)
    cam = None
    ext, mat, pro = p.extraction, p.matching, p.prosac
    glb = {
        "fast_threshold": (int, lambda v: setattr(ext, "fast_threshold", int(v) & 0xFF)),
        "fast_arc": (int, lambda v: setattr(ext, "fast_arc", v)),
        "harris_alpha": (float, lambda v: setattr(ext, "harris_alpha", v)),
        "harris_threshold": (float, lambda v: setattr(ext, "harris_threshold", v)),
        "harris_sigma": (float, lambda v: setattr(ext, "harris_sigma", v)),
        "top_n": (int, lambda v: setattr(ext, "top_n", v)),
        "n_d": (int, lambda v: setattr(ext, "n_d", v)),
        "brief_blur_sigma": (float, lambda v: setattr(ext, "brief_blur_sigma", v)),
        "patch_half": (int, lambda v: setattr(ext, "patch_half", v)),
        "lsh_tables": (int, lambda v: setattr(mat, "tables", v)),
        "lsh_bits": (int, lambda v: setattr(mat, "bits", v)),
        "lsh_probes": (int, lambda v: setattr(mat, "t_probes", v)),
        "max_distance": (int, lambda v: setattr(mat, "max_distance", v)),
        "ratio": (float, lambda v: setattr(mat, "ratio", v)),
        "prosac_threshold_px": (float, lambda v: setattr(pro, "threshold_px", v)),
        "prosac_max_iter": (int, lambda v: setattr(pro, "max_iter", v)),
        "prosac_confidence": (float, lambda v: setattr(pro, "confidence", v)),
        "homography_refresh": (int, lambda v: setattr(p, "homography_refresh", v)),
        "blend_levels": (int, lambda v: setattr(p, "blend_levels", v)),
        "seed": (int, lambda v: st.__setitem__("seed", v)),
        "overlap": (float, lambda v: st.__setitem__("overlap", v)),
        "frames_in_flight": (int, lambda v: st.__setitem__("frames_in_flight", v)),
        "workers_per_stage": (int, lambda v: st.__setitem__("workers_per_stage", v)),
    }
    for lineno, raw in enumerate(open(path), 1):
        line = raw.strip()
        if "#" in line:
            line = line[:line.index("#")].strip()
        if not line:
            continue
        if line == "[camera]":
            cams.append(dict(id=len(cams), frames=None, pre_transform=None, crop=None))
            cam = cams[-1]
            continue
        if line.startswith("["):
            raise ConfigError("ParseError", f"line {lineno}: unknown section {line}")
        if "=" not in line:
            raise ConfigError("ParseError", f"line {lineno}: expected key = value")
        key, value = (t.strip() for t in line.split("=", 1))
        if not key or not value:
            raise ConfigError("ParseError", f"line {lineno}: expected key = value")
        if cam is not None:
            if key == "id":
                cam["id"] = _num(int, value, lineno, key)
            elif key == "frames":
                cam["frames"] = value
            elif key == "pre_transform":
                v = [_num(float, t.strip(), lineno, key) for t in value.split(",")]
                if len(v) != 9:
                    raise ConfigError("ValidationError", "pre_transform: expected 9 comma-separated values")
                cam["pre_transform"] = np.array(v).reshape(3, 3)
            elif key == "crop":
                v = [_num(float, t.strip(), lineno, key) for t in value.split(",")]
                if len(v) != 4:
                    raise ConfigError("ValidationError", "crop: expected x0,y0,x1,y1")
                cam["crop"] = tuple(int(x) for x in v)
            else:
                raise ConfigError("ValidationError", f"unknown camera key: {key}")
            continue
        if key == "output_dir":
            st["output_dir"] = value
        elif key == "mode":
            if value not in ("serial", "pipelined"):
                raise ConfigError("ValidationError", "mode: expected serial or pipelined")
            st["mode"] = value
        elif key == "emit_timings":
            st["emit_timings"] = value in ("true", "1")
        elif key in glb:
            kind, setter = glb[key]
            setter(_num(kind, value, lineno, key))
        else:
            raise ConfigError("ValidationError", f"unknown key: {key}")
    if st["overlap"] <= 0.0:
        raise ConfigError("ValidationError", "overlap: NoOverlap, must be > 0")
    if st["overlap"] > 1.0:
        raise ConfigError("ValidationError", "overlap: must be <= 1")
    if st["frames_in_flight"] < 1:
        raise ConfigError("ValidationError", "frames_in_flight: must be >= 1")
    if st["workers_per_stage"] < 1:
        raise ConfigError("ValidationError", "workers_per_stage: must be >= 1")
    if p.homography_refresh < 1:
        raise ConfigError("ValidationError", "homography_refresh: must be >= 1")
    if p.blend_levels < 1:
        raise ConfigError("ValidationError", "blend_levels: must be >= 1")
    p.seed = st["seed"]
    p.matching.seed = st["seed"]
    p.prosac.seed = st["seed"]
    p.overlap_fraction = st["overlap"]
    for c in cams:
        c["files"] = []
        if c["frames"]:
            c["files"] = sorted(glob.glob(c["frames"]))
            if not c["files"]:
                raise ConfigError("MissingFrames", f"no files match pattern: {c['frames']}")
    return p, cams, st


def _log(msg):
    print(msg, file=sys.stderr)


def cmd_stitch(lp, p, cams, st):
    """cmd_stitch (cli.hpp:89-176) on the device rig."""
    if len(cams) < 2:
        _log("error: stitch needs at least 2 cameras")
        return 2
    for c in cams:
        if not c["files"]:
            _log(f"error: camera {c['id']} has no frames")
            return 2
    nframes = min(len(c["files"]) for c in cams)
    os.makedirs(st["output_dir"], exist_ok=True)
    first = [load_pnm(c["files"][0]) for c in cams]
    if any(f.ndim != 2 for f in first):
        _log("error: fast_corners: grayscale input required")
        return 1
    h, w = first[0].shape
    layout = [(c["pre_transform"], c["crop"]) for c in cams]
    use_layout = any(t is not None or cr is not None for t, cr in layout)
    rig = Rig(lp, len(cams), w, h, p, cameras=layout if use_layout else None)
    rig.set_egress_rgb(True)
    cap = rig.panorama_capacity()
    rows, stage_ns = [], [[] for _ in STAGES]
    pano = np.empty(cap, np.uint8)
    fo = abi.FrameOut()
    fo.panorama = pano.ctypes.data_as(abi.c_u8p)
    fo.pano_cap = cap
    t0 = time.perf_counter()
    done = 0
    for f in range(nframes):
        t_in = time.perf_counter_ns()
        imgs = first if f == 0 else [load_pnm(c["files"][f]) for c in cams]
        t_ing = time.perf_counter_ns() - t_in
        try:
            rig.stitch_raw([i.ctypes.data for i in imgs], f, fo)
        except abi.LorbError as e:
            _log(f"error: dropped frame {f}: {e}")
            continue
        cv = fo.canvas
        t_o = time.perf_counter_ns()
        save_pnm(os.path.join(st["output_dir"], f"pano_{f}.ppm"),
                 pano[:3 * cv.width * cv.height].reshape(cv.height, cv.width, 3))
        t_out = time.perf_counter_ns() - t_o
        dev = [float(x) for x in fo.stage_ms]
        per = [t_ing, 0.0, dev[0] * 1e6, dev[1] * 1e6, dev[2] * 1e6, dev[3] * 1e6, t_out]
        for s, ns in enumerate(per):
            stage_ns[s].append(ns)
            rows.append(f"{f},{STAGES[s]},{int(ns)}")
        done += 1
    wall = time.perf_counter() - t0
    if st["emit_timings"]:
        with open(os.path.join(st["output_dir"], "timings.csv"), "w") as out:
            out.write("frame_index,stage,duration_ns\n")
            for r in rows:
                out.write(r + "\n")
            for s, name in enumerate(STAGES):
                v = sorted(stage_ns[s]) or [0.0]
                p50 = v[len(v) // 2]
                p99 = v[min(len(v) - 1, int(math.ceil(0.99 * len(v))) - 1)]
                out.write(f"summary,{name},{np.mean(v):.0f},{p50:.0f},{p99:.0f}\n")
    print(f"frames in/out: {nframes}/{done}  throughput: {done / max(wall, 1e-9):.2f} fps  wall: {wall:.2f}s")
    rig.close()
    return 0 if done >= 1 else 1


def cmd_extract(lp, p, st, image_path):
    """cmd_extract (cli.hpp:177-207): features.csv of one image, full-image region."""
    img = load_pnm(image_path)
    if img.ndim != 2:
        _log("error: fast_corners: grayscale input required")
        return 1
    ph = p.extraction.patch_half
    h, w = img.shape
    pairs = lp.brief_pattern(p.extraction.n_d, ph, p.seed)
    try:
        kps, desc = lp.extract_features(img, [(ph, ph, w - ph, h - ph, 0)], p.extraction, pairs)
    except abi.LorbError as e:
        _log(f"error: {e}")
        return 1
    os.makedirs(st["output_dir"], exist_ok=True)
    W = (p.extraction.n_d + 63) // 64
    with open(os.path.join(st["output_dir"], "features.csv"), "w") as out:
        out.write("x,y,response,region_id,gt_plane,lt_plane\n")
        for k, d in zip(kps, desc):
            resp = np.int32(k[2]).view(np.float32)
            gt = "".join(f"{int(x):016x}" for x in d[:W])
            lt = "".join(f"{int(x):016x}" for x in d[W:2 * W])
            out.write(f"{int(k[0])},{int(k[1])},{float(resp):.6g},{int(k[3])},{gt},{lt}\n")
    _log(f"wrote {len(kps)} features")
    return 0


def _median(v):
    return sorted(v)[len(v) // 2]


def _texture(w, h, seed, sigma=1.5):
    rng = np.random.default_rng(seed)
    noise = rng.integers(0, 256, size=(h, w)).astype(np.float32)
    r = int(np.ceil(3 * sigma))
    x = np.arange(-r, r + 1, dtype=np.float32)
    k = np.exp(-(x * x) / (2 * sigma * sigma))
    k /= k.sum()
    pad = np.pad(noise, ((0, 0), (r, r)), mode="edge")
    t = sum(k[i] * pad[:, i:i + w] for i in range(2 * r + 1))
    pad = np.pad(t, ((r, r), (0, 0)), mode="edge")
    b = sum(k[i] * pad[i:i + h, :] for i in range(2 * r + 1))
    lo, hi = b.min(), b.max()
    return np.clip(np.round((b - lo) * (255.0 / (hi - lo))), 0, 255).astype(np.uint8)


def bench_features(lp, p, st, csv):
    """features_suite (cli.hpp:222-253): full-frame vs overlap-region extraction."""
    csv.write("width,height,full_ms,region_ms,ratio\n")
    ph = p.extraction.patch_half
    pairs = lp.brief_pattern(p.extraction.n_d, ph, p.seed)
    for w, h in ((800, 600), (1920, 1080), (2304, 1728)):
        img = _texture(w, h, p.seed + w)
        strip = int(math.floor(w * (1.0 - st["overlap"]) + 0.5))
        full, region = [(ph, ph, w - ph, h - ph, 0)], [(strip + ph, ph, w - ph, h - ph, 0)]
        fm, rm = [], []
        for _ in range(5):
            t = time.perf_counter()
            lp.extract_features(img, full, p.extraction, pairs)
            fm.append((time.perf_counter() - t) * 1e3)
            t = time.perf_counter()
            lp.extract_features(img, region, p.extraction, pairs)
            rm.append((time.perf_counter() - t) * 1e3)
        f, r = _median(fm), _median(rm)
        csv.write(f"{w},{h},{f:.2f},{r:.2f},{r / f:.3f}\n")
        print(f"features {w}x{h}: full {f:.1f}ms, region {r:.1f}ms, ratio {r / f:.3f}")


def bench_match(lp, p, st, csv):
    """match_suite (cli.hpp:255-299): LSH recall of perturbed queries against
    brute force over 1000 random ternary descriptors, both on the device."""
    n, queries, n_d = 1000, 100, p.extraction.n_d
    W = (n_d + 63) // 64
    rng = np.random.default_rng(p.seed)
    trits = rng.integers(-1, 2, size=(n, n_d))
    base = _pack(trits, W)
    targets = rng.integers(0, n, size=queries)
    qt = trits[targets].copy()
    for q in range(queries):
        for i in rng.integers(0, n_d, size=8):
            qt[q, i] = 1 if qt[q, i] == 0 else 0
    qd = _pack(qt, W)
    t = time.perf_counter()
    best = np.array([int(np.argmin(lp.descriptor_distances(np.repeat(qd[q:q + 1], n, 0), base, n_d)))
                     for q in range(queries)])
    brute_ms = (time.perf_counter() - t) * 1e3
    cfg = p.matching
    t = time.perf_counter()
    m = lp.match_features(qd, base, n_d, cfg)
    lsh_ms = (time.perf_counter() - t) * 1e3
    hit = {int(r[0]): int(r[1]) for r in m}
    recall = sum(1 for q in range(queries) if hit.get(q, -1) == best[q]) / queries
    csv.write("queries,recall,lsh_ms_total,brute_ms_total\n")
    csv.write(f"{queries},{recall:.3f},{lsh_ms:.2f},{brute_ms:.2f}\n")
    print(f"match: recall {recall:.3f}, lsh {lsh_ms:.2f}ms vs brute {brute_ms:.2f}ms over {queries} queries")


def _pack(trits, W):
    n, n_d = trits.shape
    out = np.zeros((n, 2 * W), np.uint64)
    for i in range(n_d):
        w, b = divmod(i, 64)
        out[:, w] |= (trits[:, i] > 0).astype(np.uint64) << np.uint64(b)
        out[:, W + w] |= (trits[:, i] < 0).astype(np.uint64) << np.uint64(b)
    return out


def bench_pipeline(lp, p, st, csv):
    """pipeline_suite (cli.hpp:301-358): 320x240 synthetic rigs of 2..7
    cameras, serial (one frame at a time) and with 1/2/4/8 frames in flight."""
    csv.write("cameras,frames_in_flight,mode,fps\n")
    frames, w, h = 20, 320, 240
    for ncams in range(2, 8):
        shift = int(math.floor(w * (1.0 - st["overlap"]) + 0.5))
        wide = _texture(w + shift * (ncams - 1), h, p.seed)
        cams = [np.ascontiguousarray(wide[:, c * shift:c * shift + w]) for c in range(ncams)]
        q = abi.Params.from_buffer_copy(p)
        q.overlap_fraction = st["overlap"]
        rig = Rig(lp, ncams, w, h, q)
        cap = rig.panorama_capacity()
        panos = [np.empty(cap, np.uint8) for _ in range(8)]
        ptrs = [c.ctypes.data for c in cams]
        for mode, fif in (("serial", 1), ("pipelined", 1), ("pipelined", 2), ("pipelined", 4), ("pipelined", 8)):
            t = time.perf_counter()
            tickets = []
            for f in range(frames):
                tickets.append(rig.submit(ptrs, f, panos[f % 8].ctypes.data, cap))
                if len(tickets) >= fif:
                    rig.wait(tickets.pop(0))
            for tk in tickets:
                rig.wait(tk)
            fps = frames / (time.perf_counter() - t)
            csv.write(f"{ncams},{fif},{mode},{fps:.2f}\n")
            print(f"pipeline cams={ncams} {mode} fif={fif}: {fps:.2f} fps")
        rig.close()


def main(argv=None):
    ap = argparse.ArgumentParser(prog="lorbpano", description="panoramic video stitching toolkit (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(sp):
        sp.add_argument("--config")
        sp.add_argument("--mode")
        sp.add_argument("--seed", type=int)
        sp.add_argument("--frames-in-flight", type=int, default=0)
        sp.add_argument("--out")
        sp.add_argument("--emit-timings", action="store_true")
        sp.add_argument("--device", type=int, default=0)
    common(sub.add_parser("stitch", help="stitch frame sequences to panoramas"))
    ex = sub.add_parser("extract", help="extract features from one image")
    common(ex)
    ex.add_argument("image")
    bp = sub.add_parser("bench", help="run a benchmark suite")
    common(bp)
    bp.add_argument("suite", nargs="?", default="features")
    a = ap.parse_args(argv)
    lp = Lorb(a.device)
    try:
        if a.config:
            p, cams, st = parse_config(a.config, lp)
        else:
            p, cams = lp.default_params(), []
            st = dict(overlap=0.25, output_dir="out", mode="serial", frames_in_flight=4, emit_timings=False, seed=0)
            p.seed = p.matching.seed = p.prosac.seed = 0
        if a.mode:
            if a.mode not in ("serial", "pipelined"):
                raise ConfigError("ValidationError", "mode: expected serial or pipelined")
            st["mode"] = a.mode
        if a.seed is not None:
            p.seed = p.matching.seed = p.prosac.seed = a.seed
        if a.frames_in_flight > 0:
            st["frames_in_flight"] = a.frames_in_flight
        if a.out:
            st["output_dir"] = a.out
        if a.emit_timings:
            st["emit_timings"] = True
    except ConfigError as e:
        _log(f"error: {e}")
        return 2
    if a.cmd == "stitch":
        if not a.config:
            _log("error: stitch requires --config")
            return 2
        return cmd_stitch(lp, p, cams, st)
    if a.cmd == "extract":
        return cmd_extract(lp, p, st, a.image)
    suites = {"features": bench_features, "match": bench_match, "pipeline": bench_pipeline}
    if a.suite not in suites:
        _log(f"error: unknown bench suite: {a.suite} (features|match|pipeline)")
        return 2
    os.makedirs(st["output_dir"], exist_ok=True)
    with open(os.path.join(st["output_dir"], f"bench_{a.suite}.csv"), "w") as csv:
        suites[a.suite](lp, p, st, csv)
    return 0


if __name__ == "__main__":
    sys.exit(main())
