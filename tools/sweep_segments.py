"""Judge time versus segments per stream (work-item granularity) on a bench
workload, to calibrate capi.cu's choose_segments.  Outputs are checked to be
identical for every S.

    python tools/sweep_segments.py c4 1,2,3,4,6,8,12,16
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200 import _lib  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge, collect_timing, set_profiling  # noqa: E402


def main():
    name = sys.argv[1]
    segs = [int(x) for x in sys.argv[2].split(",")]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    wl = bench.WORKLOADS[name]
    F, H, W = wl.frames, wl.height, wl.width
    vol = bench.make_frames(wl, range(F), os.cpu_count() or 1)
    frames = torch.from_numpy(vol).cuda()
    lib = _lib.load()
    ref = None
    for S in [0] + segs:
        lib.pcbz_set_segment_override(S)
        judge = DeviceJudge((F, H, W), (wl.pitch, wl.pitch), wl.codes, temporal=wl.temporal)
        judge(frames)
        torch.cuda.synchronize()
        set_profiling(True)
        collect_timing()
        for _ in range(steps):
            judge(frames)
        torch.cuda.synchronize()
        h, t, _ = collect_timing()
        set_profiling(False)
        out = (judge.sel.clone(), judge.ent.clone())
        if ref is None:
            ref = out
        same = torch.equal(out[0], ref[0]) and torch.equal(torch.nan_to_num(out[1]), torch.nan_to_num(ref[1]))
        print(json.dumps({"workload": name, "segments": S or "auto", "judge_ms": t / steps,
                          "hist_ms": h / steps, "GBps_raw": F * 2 * H * W / (t / steps * 1e-3) / 1e9,
                          "identical": same}), flush=True)
    lib.pcbz_set_segment_override(0)


if __name__ == "__main__":
    main()
