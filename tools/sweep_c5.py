"""Config C5 (BASELINE.json configs[4]): judge-stage throughput versus work
granule ("block size": segments per (frame, candidate) stream, from whole
frames down to a few macro-pixel rows per CTA) and versus candidate count K.

    python tools/sweep_c5.py [nframes]     -> one JSON line per point, plus a
                                              parity check that every granule
                                              gives identical entropies/modes

Granule: a stream of H*W pixels split into S segments, one CTA per segment,
192 contiguous lane runs per CTA; S = 1 is one whole frame per CTA, large S
approaches one lenslet row (15 pixel rows x 2048) per lane run.
"""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from workloads.configs import _gen_one  # noqa: E402
from paper_2310_09467_b200 import _lib  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge, collect_timing, set_profiling  # noqa: E402


def timed(judge, frames, steps=3):
    judge(frames)
    torch.cuda.synchronize()
    set_profiling(True)
    collect_timing()
    for _ in range(steps):
        judge(frames)
    torch.cuda.synchronize()
    h, t, _ = collect_timing()
    set_profiling(False)
    return h / steps, t / steps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    params = bench.c2_params()
    pick = [params[i] for i in np.linspace(0, len(params) - 1, n).astype(int)]
    with ProcessPoolExecutor(os.cpu_count() or 1) as ex:
        vol = np.stack(list(ex.map(_gen_one, pick)))
    frames = torch.from_numpy(vol).cuda()
    raw = vol.nbytes
    lib = _lib.load()
    ref_sel = ref_ent = None
    for S in (1, 2, 4, 8, 16, 32, 64, 128):
        lib.pcbz_set_segment_override(S)
        judge = DeviceJudge(vol.shape, (15, 15), list(range(13)), temporal=False, want_hist=False)
        h, t = timed(judge, frames)
        ent, sel = judge.ent.cpu().numpy(), judge.sel.cpu().numpy()
        if ref_sel is None:
            ref_sel, ref_ent = sel, ent
        same = bool(np.array_equal(sel, ref_sel) and np.array_equal(ent, ref_ent))
        print(json.dumps({"sweep": "granule", "segments_per_stream": S,
                          "pixels_per_lane_run": 2048 * 2048 // (S * 192), "candidates": 13,
                          "judge_ms": t, "hist_ms": h, "GBps_raw": raw / (t * 1e-3) / 1e9,
                          "outputs_identical_to_S1": same}), flush=True)
    lib.pcbz_set_segment_override(0)
    for K in (1, 2, 4, 8, 13, 26):
        codes = list(range(13))[:K] if K <= 13 else list(range(13)) + [0x80 | i for i in range(13)]
        if K < 13:
            codes = [0, 1, 5, 9, 12, 3, 7, 11][:K] if K <= 8 else codes
        temporal = K > 13
        if temporal:  # consecutive C2 frames stand in for a series here (timing only)
            judge = DeviceJudge(vol.shape, (15, 15), codes, temporal=True)
        else:
            judge = DeviceJudge(vol.shape, (15, 15), codes, temporal=False)
        h, t = timed(judge, frames)
        print(json.dumps({"sweep": "candidates", "K": K, "codes": codes, "judge_ms": t, "hist_ms": h,
                          "GBps_raw": raw / (t * 1e-3) / 1e9,
                          "events_per_s": (sum(K if (f > 0 or not temporal) else 13 for f in range(n))
                                           * 2 * 2048 * 2048) / (h * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
