"""Profiling driver for the emission kernel: judge + emit of 100 C2 frames
(device-resident).  Used under ncu with -k regex:emit_chunks."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2310_09467_b200.device import DeviceJudge  # noqa: E402
from workloads.configs import WORKLOADS, make_frames  # noqa: E402

wl = WORKLOADS["c2"]
vol = make_frames(wl, range(100), os.cpu_count() or 1)
frames = torch.from_numpy(vol).cuda()
judge = DeviceJudge(vol.shape, (15, 15), wl.codes, temporal=False)
for _ in range(2):
    judge(frames)
torch.cuda.synchronize()
