"""Pinned host<->device copy bandwidth of this box (the end-to-end bench's link)."""
import time
import torch
n = 33_177_600
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    print(f"{name} {50 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"both directions at once: {2 * 50 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s total")

# the same volumes split across several streams (one copy engine each?)
for nsplit in (2, 4):
    hs = [torch.empty(n // nsplit, dtype=torch.uint8).pin_memory() for _ in range(nsplit)]
    ds = [torch.empty(n // nsplit, dtype=torch.uint8, device="cuda") for _ in range(nsplit)]
    hs2 = [torch.empty(n // nsplit, dtype=torch.uint8).pin_memory() for _ in range(nsplit)]
    ds2 = [torch.empty(n // nsplit, dtype=torch.uint8, device="cuda") for _ in range(nsplit)]
    ss = [torch.cuda.Stream() for _ in range(2 * nsplit)]
    for name, both in (("H2D", False), ("H2D+D2H", True)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(50):
            for i in range(nsplit):
                with torch.cuda.stream(ss[i]):
                    ds[i].copy_(hs[i], non_blocking=True)
                if both:
                    with torch.cuda.stream(ss[nsplit + i]):
                        hs2[i].copy_(ds2[i], non_blocking=True)
        torch.cuda.synchronize()
        vol = (2 if both else 1) * 50 * (n // nsplit) * nsplit
        print(f"{name} split over {nsplit} streams: {vol / (time.perf_counter() - t) / 1e9:.1f} GB/s")
