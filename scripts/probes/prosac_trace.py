"""cfg1 frames through a PROSAC-trace build (LPB_LIB=build/variants/ptrace/...): phase deltas of pair 0."""
import os, sys, subprocess
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
if len(sys.argv) < 2:
    out = subprocess.run([sys.executable, __file__, "run"], capture_output=True, text=True).stdout
    rows = [l.split() for l in out.splitlines() if l.startswith("PT ")]
    sw = [l.split()[1] for l in out.splitlines() if l.startswith("PT-sweeps")]
    print("jacobi sweeps (block 0, warp 0):", " ".join(sw[-8:]))
    frames, cur = [], []
    for _, tag, t in rows:
        if tag == "start" and cur:
            frames.append(cur); cur = []
        cur.append((tag, int(t)))
    frames.append(cur)
    for f in frames[-2:]:
        t0 = f[0][1]
        print(" ".join(f"{tag}+{(t - p) / 1e3:.1f}" for (tag, t), (_, p) in zip(f[1:], f[:-1]))
              + f"  total {(f[-1][1] - t0) / 1e3:.1f} us")
    sys.exit(0)
from oracle import Oracle
from paper_1810_03988_b200 import Lorb
orc = Oracle("orc"); lp = Lorb(0); p = lp.default_params(); p.seed = 42; p.matching.seed = 42
l, r, _ = orc.planted_pair(int(os.environ.get("W", 640)), int(os.environ.get("H", 480)), 0.25, 42)
for i in range(4):
    lp.stitch_frame([l, r], p, frame_index=0)
