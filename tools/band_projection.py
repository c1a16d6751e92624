"""Per-rank cost of within-frame band sharding, measured on ONE GPU.

For N bands, each band's partial judge (pcbz_judge_band_device) is timed
alone -- what rank b would run -- plus the merge (finalize + argmin, run by
every rank) and one band's emission.  No rank waits on another (the bands run
as separate, independent launches), so this is a measurement of per-rank
compute, not an emulation of the collective; the collective's payload (sum
of K x 256 KiB histograms per frame, gather of the segment summaries) is
reported in bytes.

    python tools/band_projection.py [c4|c1] [steps]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200.device import BandJudge, DeviceJudge  # noqa: E402


def timed(fn, steps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    wl = bench.WORKLOADS[name]
    F, H, W = wl.frames, wl.height, wl.width
    import os
    vol = bench.make_frames(wl, range(F), os.cpu_count() or 1)
    frames = torch.from_numpy(vol).cuda()
    pitch = (wl.pitch, wl.pitch)
    whole = DeviceJudge((F, H, W), pitch, wl.codes, temporal=wl.temporal)
    t_whole = timed(lambda: whole(frames), steps)
    sel_ref = whole.sel.clone()
    raw = F * 2 * H * W
    print(json.dumps({"workload": name, "mode": "whole frames, one GPU", "ms": t_whole,
                      "GBps_raw": raw / (t_whole * 1e-3) / 1e9}), flush=True)
    for n in (1, 2, 4, 8):
        judges = [BandJudge((F, H, W), pitch, wl.codes, wl.temporal, False, b, n) for b in range(n)]
        part = [timed(lambda j=j: j.partial(frames), steps) for j in judges]
        # collective stand-in (sum + band-ordered copy) so the merge sees real inputs
        total = sum(j.hist for j in judges[1:]) + judges[0].hist if n > 1 else judges[0].hist
        judges[0].hist.copy_(total)
        for j in judges:
            judges[0].summaries[j.band].copy_(j.summary)
        t_merge = timed(lambda: judges[0].merge(), steps)
        if not torch.equal(judges[0].sel, sel_ref):
            raise RuntimeError(f"band-merged modes differ from the whole-frame judge (N={n})")
        for j in judges:
            j.sel.copy_(judges[0].sel)
        t_emit = max(timed(lambda j=j: j.emit(frames), steps) for j in judges)
        per_rank = max(part) + t_merge + t_emit
        print(json.dumps({
            "workload": name, "bands": n, "partial_ms_per_band": part, "merge_ms": t_merge,
            "emit_ms_max_band": t_emit, "per_rank_compute_ms": per_rank,
            "allreduce_bytes": judges[0].hist.numel() * 4,
            "allgather_bytes_per_rank": judges[0].summary.numel() * 2,
            "GBps_raw_excluding_collective": raw / (per_rank * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
