#!/usr/bin/env python
"""Upper bound for overlapping consecutive frames' compositors: N independent
config-3 rigs (own streams, own arenas) driven from N host threads on one GPU,
device-resident inputs; prints aggregate frames/s for N = 1..4.
usage: concurrent_rigs.py [steps]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import make_frame_sets  # noqa: E402
from paper_1810_03988_b200 import Lorb, Rig, frame_out  # noqa: E402


def main(steps=100):
    lp = Lorb(0)
    p = lp.default_params()
    p.seed = p.matching.seed = 42
    p.homography_refresh = 1 << 30
    sets, _ = make_frame_sets(4, 3840, 2160, 4)
    dev = [[torch.from_numpy(c).cuda() for c in s] for s in sets]
    for n in (1, 2, 3, 4):
        rigs = [Rig(lp, 4, 3840, 2160, p) for _ in range(n)]
        outs = [torch.empty(r.panorama_capacity(), dtype=torch.uint8, device="cuda") for r in rigs]
        fos = [frame_out(o.data_ptr(), o.numel()) for o in outs]

        def run(i, k, base):
            for t in range(k):
                rigs[i].stitch_raw([x.data_ptr() for x in dev[(t + i) % len(dev)]], base + t, fos[i])
            torch.cuda.synchronize()
        ths = [threading.Thread(target=run, args=(i, 5, 0)) for i in range(n)]
        [t.start() for t in ths]
        [t.join() for t in ths]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ths = [threading.Thread(target=run, args=(i, steps, 100)) for i in range(n)]
        [t.start() for t in ths]
        [t.join() for t in ths]
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        print(f"rigs={n} aggregate {n * steps / el:.1f} frames/s", flush=True)
        for r in rigs:
            r.close()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
