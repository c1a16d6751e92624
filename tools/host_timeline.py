"""Per-chunk timeline of the pipelined host API (pcbz_judge_host) on a C2-like
batch: PCBZ_HOST_TRACE=1 makes the library print, for every chunk, when its
upload, judge and download finished (ms after the first upload).

    python tools/host_timeline.py [nframes]      (env PCBZ_HOST_CHUNK / PCBZ_HOST_RAMP to sweep)
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PCBZ_HOST_TRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads.configs as wc  # noqa: E402
import workloads.configs as wc  # noqa: E402
from paper_2310_09467_b200 import pipeline  # noqa: E402
from paper_2310_09467_b200.core import LensletGeometry  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
params = bench.frame_params()[:n]
from concurrent.futures import ProcessPoolExecutor  # noqa: E402
with ProcessPoolExecutor(os.cpu_count() or 1) as ex:
    vol = np.stack(list(ex.map(wc._gen_one, params)))
H, W = vol.shape[1:]
pinned = torch.empty(vol.shape, dtype=torch.uint16).pin_memory()
pinned.numpy()[...] = vol
vol_np = pinned.numpy()
codes = list(range(13))
ent = torch.empty((n, 13), dtype=torch.float64).pin_memory().numpy()
sel = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
st = torch.empty((n, 2 * H * W), dtype=torch.uint8).pin_memory().numpy()
geo = LensletGeometry(15, 15)
for i in range(3):
    t0 = time.perf_counter()
    pipeline.judge_volume(vol_np, geo, codes, False, out=(ent, sel, st))
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt * 1e3:.2f} ms wall, {vol.nbytes / dt / 1e9:.1f} GB/s", file=sys.stderr, flush=True)
