"""PCIe bandwidth of pinned copies on this box (the e2e bound of
pcbz_judge_host): H2D, D2H, both at once, and each split over 2 / 4
concurrent streams (copy engines).  python tools/pcie_bw.py"""
import time

import torch

n = 839 * 2**20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best


def split(dst, src, parts, base):
    step = n // parts
    for i in range(parts):
        with torch.cuda.stream(streams[base + i]):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)


for parts in (1, 2, 4):
    for name, f in [("h2d", lambda: split(d1, h1, parts, 0)), ("d2h", lambda: split(h2, d2, parts, 4)),
                    ("both", lambda: (split(d1, h1, parts, 0), split(h2, d2, parts, 4)))]:
        s = t(f)
        print(f"{parts} stream(s) {name}: {s * 1e3:.2f} ms, {n / s / 1e9:.1f} GB/s per direction", flush=True)
