#!/usr/bin/env python
"""Benchmark: stitched panorama frames/sec on B200 (BASELINE.json metric).

Workload (default, BASELINE config 3): a 4-camera chain of 3840x2160 grayscale
frames with 25% overlap, cached homographies (estimated on the first frame,
homography_refresh = 2^30) and per-frame detect + describe + warp/blend, as
the reference's StitchEngine runs it (pipeline.hpp:645-658). One step = one
stitched frame. Inputs are synthetic: synth::texture (synth.hpp:17-34, the
reference's own generator, byte-identical through lp_synth_texture), eight
distinct frame sets rotate so the per-step input stream (8 x 33 MB) exceeds
the 126 MB L2.

N GPUs (torchrun): one independent rig per GPU (weak scaling, no collective on
the data path); an NCCL all_reduce(MAX) of the per-rank device times and an
all_gather of per-rank checksums are the only collectives.

--impl reference: the reference's own CPU engine (oracle/_ref, the unmodified
reference headers compiled here), serial engines on all host threads.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stitched panorama frames/sec (4K, 4-cam) at 1/2/4/8 B200; per-stage ms; HBM GB/s vs peak"

CONFIGS = {
    "cfg3": dict(ncams=4, w=3840, h=2160, refresh=1 << 30,
                 workload="cfg3: 4-camera 3840x2160 chain, cached homographies, per-frame "
                          "detect+describe+warp+multi-band blend"),
    "cfg4": dict(ncams=8, w=3840, h=2160, refresh=1,
                 workload="cfg4: 8-camera 3840x2160 chain, full per-frame L-ORB/LSH/PROSAC "
                          "re-registration + warp + multi-band blend"),
    "cfg2": dict(ncams=2, w=1920, h=1080, refresh=1,
                 workload="cfg2: 2-camera 1920x1080, per-frame re-registration"),
    "cfg1": dict(ncams=2, w=640, h=480, refresh=1,
                 workload="cfg1: 2-camera 640x480 planted pair, full pipeline"),
    "cfg5": dict(ncams=2, w=1920, h=1080, refresh=1, streams=64,
                 workload="cfg5: 64 independent 1920x1080 2-camera streams, per-frame "
                          "re-registration, sharded contiguously across the GPUs"),
}


def run_streams(args, cfgd, lp, world, rank, local, dist):
    """Config 5: the rank's contiguous share of 64 independent 2-camera streams
    (one rig each), driven by host threads, each keeping up to LPB_CFG5_DEPTH
    frames of each of its rigs in flight. A step = one frame of every stream
    of the job."""
    import threading

    import torch

    from paper_1810_03988_b200 import Rig, kernel_launches, load
    from paper_1810_03988_b200.shard import RankResult, aggregate_fps, gather_results, shard_streams
    lib = load()
    mine = shard_streams(cfgd["streams"], world, rank)
    p = lp.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = cfgd["refresh"]
    w, h = cfgd["w"], cfgd["h"]
    rigs, host_in, inputs, panos = [], [], [], []
    for s in mine:
        sets, _ = make_frame_sets(2, w, h, 1, seed=42 + s)
        host_in.append(sets[0])
        inputs.append([torch.from_numpy(c).cuda() for c in sets[0]])
        rig = Rig(lp, 2, w, h, p)
        rigs.append(rig)
        panos.append(torch.empty(rig.panorama_capacity(), dtype=torch.uint8, device="cuda"))
    nthreads = min(len(rigs), int(os.environ.get("LPB_CFG5_THREADS", "32")))
    depth = int(os.environ.get("LPB_CFG5_DEPTH", "3"))
    groups = [list(range(i, len(rigs), nthreads)) for i in range(nthreads)]

    def run(steps, base, ins, outs):
        errs = []

        def worker(ids):
            try:
                pending = {i: [] for i in ids}
                for t in range(steps):
                    for i in ids:
                        pending[i].append(rigs[i].submit([x.data_ptr() for x in ins[i]], base + t,
                                                         outs[i][t % len(outs[i])].data_ptr(), outs[i][0].numel()))
                        if len(pending[i]) >= depth:
                            rigs[i].wait(pending[i].pop(0))
                for i in ids:
                    for tk in pending[i]:
                        rigs[i].wait(tk)
            except Exception as e:  # surfaced after join
                errs.append(e)
        ths = [threading.Thread(target=worker, args=(g,)) for g in groups]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        if errs:
            raise errs[0]

    dev_out = [[pb] + [torch.empty_like(pb) for _ in range(depth - 1)] for pb in panos]
    run(args.warmup, 0, inputs, dev_out)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = Clocks(local)
    n0 = kernel_launches()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(args.steps, 1000, inputs, dev_out)
    torch.cuda.synchronize()
    el_ms = (time.perf_counter() - t0) * 1e3
    clk = clocks.stop()
    launches = kernel_launches() - n0
    csum = sum(int(pb[:1 << 20].to(torch.int64).sum().item()) for pb in panos)
    coll_dev = torch.device("cuda", local) if dist is None or dist.get_backend() == "nccl" else torch.device("cpu")
    ms_max, frames, checksums = gather_results(RankResult(args.steps * len(rigs), el_ms, csum), coll_dev)

    # per-kernel roofline of one of the streams (device-resident frames)
    roofline, stage, stage_ms = (None, {}, None)
    if not args.no_profile:
        fo_cap = rigs[0].panorama_capacity()
        from paper_1810_03988_b200 import frame_out
        fo = frame_out(panos[0].data_ptr(), fo_cap)
        roofline, stage, stage_ms = profile_pass(
            lib, rigs[0], lambda i: rigs[0].stitch_raw([x.data_ptr() for x in inputs[0]], 20_000 + i, fo),
            max(args.steps, 50), args.config)

    # end to end: pinned host frames in, pinned host panoramas out
    e2e = None
    if not args.no_e2e:
        pin_in = [[torch.from_numpy(c).pin_memory() for c in fr] for fr in host_in]
        pin_out = [[torch.empty(pb.numel(), dtype=torch.uint8).pin_memory() for _ in range(depth)] for pb in panos]
        run(2, 40_000, pin_in, pin_out)
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        run(args.steps, 50_000, pin_in, pin_out)
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": cfgd["streams"] * args.steps / float(tt.item()), "unit": "frames/s",
               "h2d_bytes_per_step": cfgd["streams"] * 2 * w * h,
               "d2h_bytes_per_step": None,
               "timing": f"wall clock, {nthreads} host threads, {depth} frames in flight per stream, pinned "
                         "host frames in and pinned host panoramas out, max over ranks"}
        cv = rigs[0].wait(rigs[0].submit([x.data_ptr() for x in pin_in[0]], 60_000, pin_out[0][0].data_ptr(),
                                         pin_out[0][0].numel()))
        e2e["d2h_bytes_per_step"] = cfgd["streams"] * cv[0] * cv[1]

    def params_fn(o):
        q = o.default_params()
        q.seed = q.matching.seed = 42
        q.homography_refresh = cfgd["refresh"]
        return q
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = cpu_baseline(host_in[0], params_fn, 1)
        cpu["sample"] = "stream 0: " + cpu["sample"]
    if rank == 0 and world == 1:
        parity = parity_check(rigs[0], host_in[0], params_fn)

    if rank == 0:
        line = {"metric": METRIC, "value": aggregate_fps(frames, ms_max), "unit": "frames/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u8/f32/f64", "data": "synthetic",
                "config": {"workload": cfgd["workload"], "streams": cfgd["streams"],
                           "streams_per_gpu": len(mine), "host_threads_per_gpu": nthreads,
                           "frames_in_flight_per_stream": depth,
                           "cameras": 2, "width": w, "height": h,
                           "l2": "64 distinct streams (265 MB of frames) > 126 MB L2",
                           "parallelism": f"shards x{world} (contiguous stream blocks, no data-path collective)"},
                "timing": "wall clock between device-wide synchronisations, max over ranks",
                "gpu_launches": int(launches), "clocks": clk, "rank_checksums": checksums,
                "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
                "stage_ms": stage_ms, "kernel_ms": stage}
        s = json.dumps(line)
        print(s)
        if args.out:
            open(args.out, "w").write(s + "\n")
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def texture(w, h, seed, sigma=1.5):
    """synth::texture (synth.hpp:17-34), the reference's own input generator,
    through the C-ABI's host restatement (lp_synth_texture, byte-identical)."""
    from paper_1810_03988_b200.lib import synth_texture
    return synth_texture(w, h, seed, sigma)


def make_frame_sets(ncams, w, h, nsets, seed=42, overlap=0.25):
    shift = int(np.floor(w * (1 - overlap) + 0.5))
    wide = texture(w + shift * (ncams - 1), h, seed)
    sets = []
    size = max(4, h // 16)
    for s in range(nsets):
        cams = [np.ascontiguousarray(wide[:, c * shift:c * shift + w]) for c in range(ncams)]
        # a moving bright square per set (synth::sequence_frame, synth.hpp:99-115)
        px, py = (s * 7 * 37) % (w - size), (s * 3 * 37) % (h - size)
        for c in range(ncams):
            x0 = px - c * shift
            if -size < x0 < w:
                cams[c] = cams[c].copy()
                cams[c][py:py + size, max(0, x0):min(w, x0 + size)] = 255
        sets.append(cams)
    return sets, shift


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region.

    NVML (nvidia_ml_py) polled from a thread every 2 ms, so even a timed
    region of a few tens of milliseconds carries samples; nvidia-smi -lms 100
    is the fallback when NVML is unavailable."""

    def __new__(cls, index):
        try:
            return _NvmlClocks(index)
        except Exception:
            return super().__new__(cls)

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


class _NvmlClocks:
    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index):
        import threading

        import pynvml as N
        N.nvmlInit()
        self.N = N
        h = None
        try:  # map the torch device to its NVML handle through the UUID
            import torch
            u = str(torch.cuda.get_device_properties(index).uuid)
            h = N.nvmlDeviceGetHandleByUUID(u if u.startswith("GPU-") else "GPU-" + u)
        except Exception:
            h = N.nvmlDeviceGetHandleByIndex(index)
        self.h = h
        self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        self.rows = []
        self.stop_ev = threading.Event()
        self.sample()
        self.th = threading.Thread(target=self.loop, daemon=True)
        self.th.start()

    def sample(self):
        N = self.N
        sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
        rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        util = N.nvmlDeviceGetUtilizationRates(self.h).gpu
        self.rows.append((float(sm), int(rs), int(util)))

    def loop(self):
        while not self.stop_ev.wait(0.002):
            self.sample()

    def stop(self):
        self.stop_ev.set()
        self.th.join()
        self.sample()
        N = self.N
        rows = self.rows
        loaded = [r for r in rows if r[2] > 0] or rows
        reasons = sorted({name for name, attr in self.REASONS for r in rows
                          if r[1] & getattr(N, attr, 0)})
        try:
            N.nvmlShutdown()
        except Exception:
            pass
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "sampler": "NVML every 2 ms"}


def measured_peak_hbm():
    try:
        j = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def pipe_peaks():
    """Measured per-pipe peaks of this B200 (scripts/probes/pipe_peaks.cu,
    profiles/peaks_fp64_int.json) plus the HBM copy peak, in G op/s (GB/s)."""
    hbm, hbm_src = measured_peak_hbm()
    pk = {"hbm": (hbm, hbm_src)}
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64_int.json")))["peaks"]
        src = "measured (profiles/peaks_fp64_int.json, scripts/probes/pipe_peaks.cu)"
        pk["fp64"] = (j["dadd"]["Gop_s"], src)
        pk["fp64_div"] = (j["ddiv_rn"]["Gop_s"], src)
        pk["fp32"] = (j["ffma"]["Gop_s"], src)
        pk["popc"] = (j["popc"]["Gop_s"], src)
    except Exception:  # B200_PROFILING.md-style nominal fallbacks at 1965 MHz, 148 SMs
        f = 148 * 1.965
        src = "fallback (nominal per-SM rates x 148 SMs x 1965 MHz)"
        pk.update({"fp64": (64 * f, src), "fp64_div": (4 * f, src), "fp32": (128 * f, src),
                   "popc": (16 * f, src)})
    return pk


def kernel_roofline(lib, rig, key, avg_ms, launches):
    """One kernel against every pipe its algorithmic work uses; the bound is
    the pipe with the largest fraction of its peak. FP64 divisions/square
    roots are converted to add/mul slots by the measured peak ratio, so the
    FP64 figure is 'DADD-equivalent G op/s' against the DADD peak. Peaks of a
    launch that can occupy only some SMs (one cluster per camera pair) are
    scaled to those SMs."""
    w = (C.c_double * 6)()
    st = lib.lp_rig_algorithmic_work(rig, key.encode(), int(launches), w)
    pk = pipe_peaks()
    t = avg_ms * 1e-3
    occ = (w[5] / 148.0) if w[5] > 0 else 1.0
    pipes = {}
    if st == 0 and w[0] > 0:
        pipes["hbm"] = (w[0] / 1e9, pk["hbm"][0], "GB/s", pk["hbm"][1])
    if st == 0 and (w[1] > 0 or w[2] > 0):
        eq = w[1] + w[2] * pk["fp64"][0] / pk["fp64_div"][0]
        pipes["fp64"] = (eq / 1e9, pk["fp64"][0] * occ, "Gop/s (DADD-equivalent)", pk["fp64"][1])
    if st == 0 and w[3] > 0:
        pipes["fp32"] = (w[3] / 1e9, pk["fp32"][0] * occ, "Gop/s", pk["fp32"][1])
    if st == 0 and w[4] > 0:
        pipes["popc"] = (w[4] / 1e9, pk["popc"][0] * occ, "Gop/s", pk["popc"][1])
    if not pipes:
        return {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                "avg_launch_ms": avg_ms, "algorithmic": None}
    fr = {p: (v[0] / t) / v[1] for p, v in pipes.items()}
    b = max(fr, key=fr.get)
    g, peak, unit, src = pipes[b]
    return {"bound": b, "achieved": g / t, "peak": peak, "unit": unit, "frac": fr[b],
            "peak_source": src + (f", scaled to the {int(w[5])} SMs the launch occupies" if w[5] > 0 else ""),
            "avg_launch_ms": avg_ms,
            "algorithmic": {"bytes": w[0], "fp64_addmul_ops": w[1], "fp64_div_sqrt_ops": w[2],
                            "fp32_ops": w[3], "popc_ops": w[4]},
            "frac_by_pipe": {p: round(f, 4) for p, f in fr.items()}}


def profile_pass(lib, rig, step, steps, config):
    """Per-kernel device times of `steps` frames with the rig's stages
    serialised on one stream (concurrent extraction would otherwise inflate
    the compositor's kernels), every kernel set against its pipes
    (kernel_roofline), the dominant one as the line's roofline."""
    import torch
    lib.lp_rig_set_streams(rig.rig, 1)
    lib.lp_profile_reset()
    lib.lp_rig_work_reset(rig.rig)
    lib.lp_profile_enable(1)
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    cap = 256
    names = C.create_string_buffer(cap * 64)
    tot = (C.c_double * cap)()
    cnt = (C.c_longlong * cap)()
    lib.lp_profile_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    n = lib.lp_profile_read(names, 64, tot, cnt, cap)
    lib.lp_profile_enable(0)
    lib.lp_rig_set_streams(rig.rig, 2)
    kern = {}
    for i in range(min(n, cap)):
        key = names.raw[i * 64:(i + 1) * 64].split(b"\0")[0].decode()
        kern[key] = (tot[i], cnt[i])
    step_ms = sum(v[0] for v in kern.values()) / steps
    dom = max(kern, key=lambda k: kern[k][0])
    # every kernel against the pipe its exact arithmetic needs most of
    # (lp_rig_algorithmic_work: compulsory bytes, FP64 add/mul/compare,
    # FP64 div/sqrt, FP32, POPC); the bound is the pipe with the largest
    # fraction of its measured peak
    per_kernel = {k: kernel_roofline(lib, rig.rig, k, kern[k][0] / kern[k][1], kern[k][1]) for k in kern}
    # DRAM bytes of the same launch from the committed ncu --set full capture
    # (scripts/ncu_traffic.py -> profiles/ncu_traffic.json), or null
    traffic, limiter = None, None
    try:
        nj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = nj.get(config, {}).get(dom, {}).get("traffic_bytes")
        limiter = nj.get(config, {}).get(dom, {}).get("limiter")
    except Exception:
        pass
    roofline = dict(per_kernel[dom])
    roofline.update({"kernel": dom, "traffic": traffic,
                     # what ncu says bounds it (same capture): issue slots / FP64 pipe / DRAM
                     "ncu_limiter": limiter,
                     "share_of_kernel_time": kern[dom][0] / max(1e-9, sum(v[0] for v in kern.values())),
                     "kernels": {k: {"ms": round(v["avg_launch_ms"], 4), "bound": v["bound"],
                                     "frac": None if v["frac"] is None else round(v["frac"], 4)}
                                 for k, v in sorted(per_kernel.items(), key=lambda kv: -kern[kv[0]][0])}})
    stage = {k: round(v[0] / v[1], 4) for k, v in sorted(kern.items(), key=lambda kv: -kv[1][0])}
    stage["_kernel_ms_per_frame"] = round(step_ms, 4)
    # the reference's stages (pipeline.hpp:26-34), device ms per frame
    ref_stages = {"rectify_crop": ("k_rectify",), "detect": ("k_detect", "k_topn"),
                  "describe": ("k_describe",),
                  "match_estimate": ("k_lsh_keys", "k_match_query", "k_match_finalize", "k_prosac", "k_chain"),
                  "warp_blend": ("k_warp", "k_runs", "k_mask0", "k_pyr_down", "k_blend_level")}
    stage_ms = {name: round(sum(v[0] for k, v in kern.items() if k.split("/")[0] in ks) / steps, 4)
                for name, ks in ref_stages.items()}
    return roofline, stage, stage_ms


def parity_check(rig, frames, params_fn):
    """The GPU rig's panorama of `frames` at frame 0 (an estimating frame, as
    the reference engine's first) against the reference StitchEngine's."""
    import oracle
    if not oracle.ref_available():
        return None
    from oracle import Oracle
    o = Oracle("ref")
    want = o.stitch_frame(frames, params_fn(o), frame_index=0)["panorama"]
    got = rig.stitch(frames, 0)["panorama"]
    same_shape = got.shape == want.shape
    return {"equal": bool(same_shape and np.array_equal(got, want)),
            "max_abs_diff": int(np.abs(got.astype(int) - want.astype(int)).max()) if same_shape else None,
            "shape": list(got.shape), "against": "reference stitch_frame (oracle/_ref), frame 0"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(frames, params_fn, sample_frames=1, pipelined_frames=4):
    """The reference CPU engine (oracle/_ref) on a bounded sample of the same
    workload: `sample_frames` frames through the serial StitchEngine on 1 core
    (mode i), then `pipelined_frames` frames through its Pipelined mode with
    frames_in_flight 4 and workers_per_stage = #cameras (mode ii,
    pipeline.hpp:660-711). Returns (baseline dict, the serial run's panorama
    as (H, W) u8 or None): the panorama is the parity check of the GPU arm."""
    import oracle
    from oracle import Oracle
    kind = "reference" if oracle.ref_available() else "port"
    o = Oracle("ref" if kind == "reference" else "orc")
    p = params_fn(o)
    ncams = len(frames)
    h, w = frames[0].shape
    stage_names = ["ingest", "rectify_crop", "detect", "describe", "match_estimate", "warp_blend", "output"]
    pano = None
    pipelined = None
    t0 = time.perf_counter()
    if kind == "reference":
        from paper_1810_03988_b200 import abi
        arr = (C.c_void_p * ncams)(*[f.ctypes.data for f in frames])
        fps, ms = C.c_double(), (C.c_double * 7)()
        cap = ncams * w * 2 * h
        buf = np.zeros(cap, np.uint8)
        cv = abi.Canvas()
        fn = o.lib.ref_run_engine_out
        fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        st = fn(ncams, w, h, C.byref(p), arr, sample_frames, 0, 1, 1, C.byref(fps), ms,
                buf.ctypes.data, cap, C.byref(cv))
        if st:
            raise abi.LorbError(st, o.lib.ref_last_error().decode())
        value = fps.value
        serial_s = time.perf_counter() - t0
        stages = {n: round(ms[i], 2) for i, n in enumerate(stage_names)}
        pano = buf[:cv.width * cv.height].reshape(cv.height, cv.width).copy()
        if pipelined_frames > 0:
            workers = ncams
            t1 = time.perf_counter()
            st = fn(ncams, w, h, C.byref(p), arr, pipelined_frames, 1, 4, workers, C.byref(fps), ms,
                    None, 0, None)
            if st:
                raise abi.LorbError(st, o.lib.ref_last_error().decode())
            pipelined = {"value": fps.value, "unit": "frames/s", "mode": "Pipelined",
                         "frames_in_flight": 4, "workers_per_stage": workers,
                         "cores": min(os.cpu_count() or 1, 7 * workers),
                         "sample": f"{pipelined_frames} frames, {time.perf_counter() - t1:.1f} s",
                         "stage_ms": {n: round(ms[i], 2) for i, n in enumerate(stage_names)}}
    else:
        for _ in range(sample_frames):
            o.stitch_frame(frames, p)
        value = sample_frames / (time.perf_counter() - t0)
        serial_s = time.perf_counter() - t0
        stages = None
    return ({"value": value, "unit": "frames/s", "cores": 1, "kind": kind,
             "sample": f"{sample_frames} frame(s) of the same workload through the reference's "
                       f"serial StitchEngine (pipeline.hpp:645-658), {serial_s:.1f} s",
             "stage_ms": stages, "pipelined": pipelined, "cpu_model": cpu_model(),
             "host_threads": os.cpu_count()}, pano)


def run_reference(args, cfgd):
    """--impl reference: the reference's own CPU engine on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from oracle import Oracle
    from paper_1810_03988_b200 import abi
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return 0
    o = Oracle("ref")
    sets, _ = make_frame_sets(cfgd["ncams"], cfgd["w"], cfgd["h"], 1)
    frames = sets[0]
    p = o.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = cfgd["refresh"]
    ncams, w, h = cfgd["ncams"], cfgd["w"], cfgd["h"]
    ncpu = os.cpu_count() or 1
    try:
        mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):
        mem_gb = 64
    per_engine_gb = 4.0 * ncams * w * h / (3840 * 2160 * 4)  # ~4 GB for 4K x 4 cams
    threads = int(max(1, min(ncpu, mem_gb * 0.5 / max(per_engine_gb, 0.1), 32)))
    steps, warm = min(args.steps, 3), min(args.warmup, 1)
    arr = (C.c_void_p * ncams)(*[f.ctypes.data for f in frames])
    agg = C.c_double()
    for _ in range(warm):
        o.lib.ref_run_engines_parallel(ncams, w, h, C.byref(p), arr, 1, threads, C.byref(agg))
    t0 = time.perf_counter()
    for _ in range(steps):
        st = o.lib.ref_run_engines_parallel(ncams, w, h, C.byref(p), arr, 1, threads, C.byref(agg))
        if st:
            raise abi.LorbError(st, o.lib.ref_last_error().decode())
    el = time.perf_counter() - t0
    value = steps * threads / el
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": el / steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/f32/f64",
            "data": "synthetic",
            "config": {"workload": cfgd["workload"], "cameras": ncams, "width": w, "height": h,
                       "engines": threads, "frames_per_step": threads},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "reference",
                             "sample": f"{threads} serial StitchEngines in parallel, 1 frame each per step"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the reference-engine check of a stitched frame")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    # `python bench.py --gpus N` without torchrun: launch the N ranks here
    # (one process per GPU, torch.distributed.run on 127.0.0.1)
    from paper_1810_03988_b200.shard import maybe_self_launch
    rc = maybe_self_launch(os.path.abspath(__file__), sys.argv[1:], args.gpus)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args, cfgd)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LPB_RANKS_ON_ONE_GPU=1 (+ LPB_DIST_BACKEND=gloo): every rank on cuda:0, a
    # single-GPU rehearsal of the multi-rank path (tests/gpu_multirank); the
    # driver's runs use one GPU per rank over NCCL
    if os.environ.get("LPB_RANKS_ON_ONE_GPU") == "1":
        local = 0
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("LPB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # communicator log (comm init lines carry nRanks) on stderr, so
            # stdout keeps the single JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = torch.device("cuda", local) if dist is None or dist.get_backend() == "nccl" else torch.device("cpu")

    from paper_1810_03988_b200 import Lorb, Rig, abi, frame_out, kernel_launches, load
    from paper_1810_03988_b200.shard import RankResult, aggregate_fps, gather_results
    lib = load()
    lp = Lorb(local)
    if args.config == "cfg5":
        return run_streams(args, cfgd, lp, world, rank, local, dist)
    ncams, w, h = cfgd["ncams"], cfgd["w"], cfgd["h"]
    p = lp.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = cfgd["refresh"]
    nsets = int(os.environ.get("LPB_NSETS", 8 if args.config in ("cfg3", "cfg4") else 4))
    sets, shift = make_frame_sets(ncams, w, h, nsets, seed=42 + rank)
    dev_sets = [[torch.from_numpy(c).cuda() for c in s] for s in sets]
    rig = Rig(lp, ncams, w, h, p)
    stream = torch.cuda.ExternalStream(rig.stream)
    pano_cap = rig.panorama_capacity()
    dpano = torch.empty(pano_cap, dtype=torch.uint8, device="cuda")
    fo = frame_out(dpano.data_ptr(), pano_cap)
    # frames in flight in the device-resident loop: the pipelined API
    # (lp_rig_submit / lp_rig_wait, 3 in flight) for cached-homography frames,
    # lp_rig_stitch one frame at a time for re-registering ones (A/B on B200:
    # cfg3 1714 -> 1755 at 3; cfg1/cfg2/cfg4 1-4 % faster at 1)
    dev_depth = int(os.environ.get("LPB_DEV_DEPTH", "3" if args.config == "cfg3" else "1"))
    dpanos = [dpano] + [torch.empty(pano_cap, dtype=torch.uint8, device="cuda") for _ in range(dev_depth - 1)]

    def step(i):
        rig.stitch_raw([t.data_ptr() for t in dev_sets[i % nsets]], i, fo)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    canvas = (fo.canvas.width, fo.canvas.height)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident inputs, CUDA events on the rig stream
    barrier()
    clocks = Clocks(local)
    n0 = kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if dev_depth > 1:
        # the rig's pipelined API (lp_rig_submit / lp_rig_wait), device-resident
        # frames in and device panoramas out, dev_depth frames in flight
        tickets = []
        for i in range(args.steps):
            tickets.append(rig.submit([t.data_ptr() for t in dev_sets[(args.warmup + i) % nsets]],
                                      args.warmup + i, dpanos[i % dev_depth].data_ptr(), pano_cap))
            if len(tickets) >= dev_depth:
                rig.wait(tickets.pop(0))
        for tk in tickets:
            rig.wait(tk)
    else:
        for i in range(args.steps):
            step(args.warmup + i)
    e1.record(stream)
    e1.synchronize()
    barrier()
    clk = clocks.stop()
    launches = kernel_launches() - n0
    ms = e0.elapsed_time(e1)
    # the only collectives: MAX of device time, SUM of frames, gather of
    # panorama checksums (paper_1810_03988_b200.shard)
    pano = dpanos[(args.steps - 1) % dev_depth][:canvas[0] * canvas[1]] if dev_depth > 1 else dpano[:canvas[0] * canvas[1]]
    csum = int(pano.to(torch.int64).sum().item())
    ms_max, total_frames, checksums = gather_results(RankResult(args.steps, ms, csum), coll_dev)
    value = aggregate_fps(total_frames, ms_max)

    # ---- per-kernel profile pass (same workload; events around every launch)
    roofline, stage, stage_ms = (None, {}, None) if args.no_profile else \
        profile_pass(lib, rig, lambda i: step(10_000 + i), args.steps, args.config)

    # ---- end to end through the public C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        # pinned host frames in, pinned host panoramas out, 3 frames in flight
        # (lp_rig_submit / lp_rig_wait): every step's ingest copy, stages and
        # panorama egress are inside the timed region
        depth = int(os.environ.get("LPB_E2E_DEPTH", "3"))
        # each set's cameras back to back in one page-locked block (one
        # ingest copy per frame); LPB_E2E_CONTIG=0: one block per camera
        wc_blocks = []
        if os.environ.get("LPB_E2E_WC", "0") == "1":
            # write-combined page-locked blocks (lp_host_alloc_wc): written
            # once here, read only by the device's copy engine
            host_sets = []
            for st in sets[:2]:
                arr = np.ascontiguousarray(np.stack(st))
                ptr = lib.lp_host_alloc_wc(arr.nbytes)
                if not ptr:
                    raise RuntimeError("lp_host_alloc_wc failed")
                wc_blocks.append(ptr)
                C.memmove(ptr, arr.ctypes.data, arr.nbytes)
                fb = arr[0].nbytes
                host_sets.append([types.SimpleNamespace(data_ptr=(lambda q: (lambda: q))(ptr + c * fb))
                                  for c in range(len(st))])
        elif os.environ.get("LPB_E2E_CONTIG", "1") != "0":
            host_sets = []
            for st in sets[:2]:
                blk = torch.from_numpy(np.ascontiguousarray(np.stack(st))).pin_memory()
                host_sets.append([blk[c] for c in range(len(st))])
        else:
            host_sets = [[torch.from_numpy(c).pin_memory() for c in s] for s in sets[:2]]
        hpanos = [torch.empty(pano_cap, dtype=torch.uint8).pin_memory() for _ in range(depth)]

        def run_e2e(n, base):
            tickets = []
            for i in range(n):
                tickets.append(rig.submit([t.data_ptr() for t in host_sets[i % len(host_sets)]], base + i,
                                          hpanos[i % depth].data_ptr(), pano_cap))
                if len(tickets) >= depth:
                    rig.wait(tickets.pop(0))
            for tk in tickets:
                rig.wait(tk)

        run_e2e(4, 20_000)
        barrier()
        t0 = time.perf_counter()
        run_e2e(args.steps, 30_000)
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        got = hpanos[(args.steps - 1) % depth][:canvas[0] * canvas[1]].to(torch.int64).sum().item()
        for ptr in wc_blocks:
            lib.lp_host_free(ptr)
        e2e = {"value": world * args.steps / float(tt.item()), "unit": "frames/s",
               "h2d_bytes_per_step": ncams * w * h, "d2h_bytes_per_step": canvas[0] * canvas[1],
               "timing": "wall clock around lp_rig_submit/lp_rig_wait (3 frames in flight) with pinned "
                         "host frames in and pinned host panoramas out",
               "last_panorama_sum": int(got)}

    # frame-level HBM figure: SURVEY §8(d) compulsory bytes per frame (camera
    # frames in, panorama out, the overlap strips' blur crops, keypoints and
    # descriptors, and on re-registration frames the descriptors in and the
    # matches + correspondences out) at the measured frame rate
    frame_hbm = None
    if rank == 0:
        ov = 0.25
        strip = int(np.floor(w * ov + 0.5))
        ph, margin = 15, 21
        crop_l = (min(w, w - ph + margin) - max(0, w - strip + ph - margin)) * h
        crop_r = (min(w, strip - ph + margin) - max(0, ph - margin)) * h
        nreg = 2 * (ncams - 1)
        B = ncams * w * h + canvas[0] * canvas[1] + (ncams - 1) * (crop_l + crop_r) + nreg * 500 * 80
        if cfgd["refresh"] == 1:
            B += (ncams - 1) * (2 * 500 * 64 + 500 * 56)
        gbps = B * value / 1e9
        peak, peak_src = measured_peak_hbm()
        frame_hbm = {"compulsory_bytes_per_frame": B, "GBps": gbps, "frac_of_peak": gbps / peak,
                     "basis": "SURVEY 8(d) B_frame at the device frame rate"}

    cpu = None
    parity = None

    def params_fn(o):
        q = o.default_params()
        q.seed = q.matching.seed = 42
        q.homography_refresh = cfgd["refresh"]
        return q
    if rank == 0 and world == 1 and args.no_cpu_baseline and not args.no_parity:
        parity = parity_check(rig, sets[0], params_fn)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, ref_pano = cpu_baseline(sets[0], params_fn, 1)
        # parity of the measured path: the GPU rig's panorama of sets[0] at
        # frame 0 (an estimating frame, as the reference engine's first)
        # against the reference engine's panorama of the same frame
        if ref_pano is not None:
            got = rig.stitch(sets[0], 0)["panorama"]
            parity = {"equal": bool(got.shape == ref_pano.shape and np.array_equal(got, ref_pano)),
                      "max_abs_diff": int(np.abs(got.astype(int) - ref_pano.astype(int)).max())
                      if got.shape == ref_pano.shape else None,
                      "shape": list(got.shape), "against": "reference StitchEngine (oracle/_ref), frame 0 of set 0"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u8/f32/f64", "data": "synthetic",
                "config": {"workload": cfgd["workload"], "cameras": ncams, "width": w, "height": h,
                           "canvas": list(canvas), "overlap": 0.25,
                           "l2": f"{nsets} rotating input frame sets ({nsets * ncams * w * h / 1e6:.0f} MB) > 126 MB L2",
                           "parallelism": f"replicas x{world} (independent rigs, no data-path collective)",
                           "device_frames_in_flight": dev_depth},
                "gpu_launches": int(launches), "clocks": clk, "roofline": roofline,
                "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "stage_ms": stage_ms if not args.no_profile else None,
                "frame_hbm": frame_hbm, "kernel_ms": stage, "rank_checksums": checksums}
        s = json.dumps(line)
        print(s)
        if args.out:
            open(args.out, "w").write(s + "\n")
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
