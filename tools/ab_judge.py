"""A/B timing of judge-library variants on a C2-like batch (device-resident).

    PCBZ_LIB=<variant .so> python tools/ab_judge.py [nframes]
Prints one JSON line: hist-kernel ms per frame and whole-judge ms per frame."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from workloads.configs import _gen_one  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge, collect_timing, set_profiling  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 52
params = bench.frame_params()
pick = [params[i] for i in np.linspace(0, len(params) - 1, n).astype(int)]

from concurrent.futures import ProcessPoolExecutor  # noqa: E402
with ProcessPoolExecutor(os.cpu_count() or 1) as ex:
    vol = np.stack(list(ex.map(_gen_one, pick)))
frames = torch.from_numpy(vol).cuda()
judge = DeviceJudge(vol.shape, (15, 15), list(range(13)), temporal=False)
for _ in range(2):
    judge(frames)
torch.cuda.synchronize()
set_profiling(True)
collect_timing()
steps = 5
for _ in range(steps):
    judge(frames)
torch.cuda.synchronize()
h, t, _ = collect_timing()
print(json.dumps({"lib": os.environ.get("PCBZ_LIB", "default"), "frames": n,
                  "hist_ms_per_frame": h / steps / n, "judge_ms_per_frame": t / steps / n,
                  "sel": judge.sel[:8].cpu().tolist()}), flush=True)
