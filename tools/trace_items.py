"""Per-work-item timing of the judge kernel (pcbz_set_item_trace): item
durations by candidate, per-SM busy time and the tail (time between the
first SM going idle and the last one finishing).

    python tools/trace_items.py c4 [segments]
"""
import json
import os
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200 import _lib  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge  # noqa: E402


def main():
    name = sys.argv[1]
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    wl = bench.WORKLOADS[name]
    F, H, W = wl.frames, wl.height, wl.width
    vol = bench.make_frames(wl, range(F), os.cpu_count() or 1)
    frames = torch.from_numpy(vol).cuda()
    lib = _lib.load()
    lib.pcbz_set_segment_override(S)
    judge = DeviceJudge((F, H, W), (wl.pitch, wl.pitch), wl.codes, temporal=wl.temporal)
    judge(frames)
    torch.cuda.synchronize()
    lib.pcbz_set_item_trace(1)
    judge(frames)
    torch.cuda.synchronize()
    buf = np.zeros(3 * (1 << 20), np.uint64)
    seg = ctypes.c_int()
    n = lib.pcbz_item_trace(buf.ctypes.data, 1 << 20, ctypes.byref(seg))
    lib.pcbz_set_item_trace(0)
    lib.pcbz_set_segment_override(0)
    rec = buf[:3 * n].reshape(n, 3)
    sm = (rec[:, 0] >> 48).astype(int)
    t0 = (rec[:, 0] & ((1 << 48) - 1)).astype(np.int64)
    t_runs = rec[:, 1].astype(np.int64)
    t1 = rec[:, 2].astype(np.int64)
    base = (int(t1[0]) >> 48) << 48   # start stamps were truncated to 48 bits
    t0 = t0 + base
    t0 = np.where(t0 > t1, t0 - (1 << 48), t0)
    S = seg.value
    def dispatch_order(lst):  # capi.cu order_by_cost: cost class descending, stable
        def cls(b):
            i = b & 0x7F
            return (4 if b & 0x80 else 0) + (0 if i == 0 else 1 + (i - 1) // 4)
        return sorted(lst, key=lambda b: -cls(b))

    codes = sorted(wl.codes)
    listA = dispatch_order([x for x in codes if not x & 0x80] if wl.temporal else codes)
    listB = dispatch_order(codes)
    kA, kB = len(listA), len(listB)
    dur = (t1 - t0) / 1e3
    by_cand = defaultdict(list)
    for item in range(n):
        pair = item // S
        c = listA[pair] if pair < kA else listB[(pair - kA) % kB]
        by_cand[c].append(dur[item])
    start = t0.min()
    busy_end = defaultdict(int)
    for s_, e in zip(sm, t1):
        busy_end[s_] = max(busy_end[s_], e)
    ends = np.array(sorted(busy_end.values())) - start
    print(json.dumps({
        "workload": name, "segments": S, "items": int(n), "sms": len(busy_end),
        "makespan_us": float((t1.max() - start) / 1e3),
        "first_sm_idle_us": float(ends[0] / 1e3), "median_sm_end_us": float(np.median(ends) / 1e3),
        "item_us_mean": float(dur.mean()), "item_us_p10": float(np.percentile(dur, 10)),
        "runs_us_mean": float(((t_runs - t0) / 1e3).mean()),
        "after_runs_us_mean": float(((t1 - t_runs) / 1e3).mean()),
        "item_us_p90": float(np.percentile(dur, 90)),
        "by_candidate_us": {f"0x{c:02X}": round(float(np.mean(v)), 1) for c, v in sorted(by_cand.items())},
    }))


if __name__ == "__main__":
    main()
