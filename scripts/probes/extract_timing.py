"""Host-call latency of lp_extract_features, full frame vs 25% strip (acceptance criterion 8 shape)."""
import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from oracle import Oracle
from paper_1810_03988_b200 import Lorb

orc = Oracle("orc")
lp = Lorb(0)
w, h = 1280, 720
img = orc.texture(w, h, 808)
p = lp.default_params()
cfg = p.extraction
pairs = lp.brief_pattern(cfg.n_d, cfg.patch_half, 808)
ph = cfg.patch_half
full = [(ph, ph, w - ph, h - ph, 0)]
strip = [(round(w * 0.75) + ph, ph, w - ph, h - ph, 0)]
for name, src in (("host", img),):
    for rname, r in (("full", full), ("strip", strip)):
        for _ in range(5):
            lp.extract_features(src, r, cfg, pairs)
        ts = []
        for _ in range(int(os.environ.get("REPS", 50))):
            t0 = time.perf_counter()
            kp, d = lp.extract_features(src, r, cfg, pairs)
            ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort()
        print(f"{name:6s} {rname:5s} median {ts[len(ts)//2]:.3f} ms min {ts[0]:.3f} n={len(kp)}")

tf, tr = [], []
for _ in range(int(os.environ.get("REPS", 40))):
    t0 = time.perf_counter(); lp.extract_features(img, full, cfg, pairs); tf.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); lp.extract_features(img, strip, cfg, pairs); tr.append(time.perf_counter() - t0)
tf.sort(); tr.sort()
print(f"interleaved: full {tf[len(tf)//2]*1e3:.3f} strip {tr[len(tr)//2]*1e3:.3f}")
