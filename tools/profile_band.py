"""Profiling driver: one C4 band partial (pcbz_judge_band_device, band 0 of
N) after a warm-up.  Used under ncu:

    python tools/profile_band.py && ncu --set full -k regex:judge_hist -s 1 -c 1 \\
        -o gpurun_out/prof python tools/profile_band.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2310_09467_b200 import _lib  # noqa: E402
from paper_2310_09467_b200.device import BandJudge  # noqa: E402
from workloads.configs import WORKLOADS, make_frames  # noqa: E402

n = int(os.environ.get("PCBZ_PROFILE_BANDS", "8"))
seg = int(os.environ.get("PCBZ_PROFILE_SEGMENTS", "0"))
if seg:
    _lib.load().pcbz_set_segment_override(seg)
wl = WORKLOADS["c4"]
vol = make_frames(wl, range(wl.frames), os.cpu_count() or 1)
frames = torch.from_numpy(vol).cuda()
j = BandJudge(vol.shape, (wl.pitch, wl.pitch), wl.codes, wl.temporal, False, 0, n)
for _ in range(2):
    j.partial(frames)
torch.cuda.synchronize()
print("segments", j.segments)
