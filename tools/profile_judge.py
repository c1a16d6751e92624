"""Profiling driver: one warm-up and one measured launch of the judge on a
reduced C2 batch (default 12 frames, all three SNR levels).  Used under ncu:

    python tools/profile_judge.py && ncu --set full -k regex:judge_hist -s 1 -c 1 \
        -o gpurun_out/prof python tools/profile_judge.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge  # noqa: E402

n = int(os.environ.get("PCBZ_PROFILE_FRAMES", "12"))
params = bench.frame_params()
pick = [params[i] for i in np.linspace(0, len(params) - 1, n).astype(int)]
from workloads.lfm_synth import generate_array  # noqa: E402
vol = np.stack([generate_array(p)[0] for p in pick])
frames = torch.from_numpy(vol).cuda()
codes = [int(c) for c in os.environ.get("PCBZ_PROFILE_CODES", ",".join(map(str, range(13)))).split(",")]
seg = int(os.environ.get("PCBZ_PROFILE_SEGMENTS", "0"))
if seg:
    from paper_2310_09467_b200 import _lib
    _lib.load().pcbz_set_segment_override(seg)
judge = DeviceJudge(vol.shape, (15, 15), codes, temporal=False)
for _ in range(2):
    judge(frames)
torch.cuda.synchronize()
print("sel", judge.sel.cpu().numpy().tolist())
