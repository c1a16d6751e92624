"""Per-rank cost of within-frame band sharding, measured on ONE GPU.

For N bands, each band's partial judge (pcbz_judge_band_device) is timed
alone -- what rank b would run -- plus the owner-computes merge of its
1/N of the slots (pcbz_judge_merge_slots_device), the argmin and one band's
emission.  No rank waits on another (the bands run
as separate, independent launches), so this is a measurement of per-rank
compute, not an emulation of the collective; the collective's payload (reduce-scatter of the K x 256 KiB histograms per
frame, all-to-all of the segment summaries, all-gather of the entropies) is
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
from paper_2310_09467_b200.shard import emulate_band_exchange, emulate_band_peer_exchange  # noqa: E402


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
    import os as _os
    seg = int(_os.environ.get("PCBZ_BAND_SEGMENTS", "0"))
    if seg:
        from paper_2310_09467_b200 import _lib
        _lib.load().pcbz_set_segment_override(seg)
    for n in [int(x) for x in _os.environ.get("PCBZ_BAND_COUNTS", "1,2,4,8").split(",")]:
        judges = [BandJudge((F, H, W), pitch, wl.codes, wl.temporal, False, b, n) for b in range(n)]
        part = [timed(lambda j=j: j.partial(frames), steps) for j in judges]
        emulate_band_exchange(judges)          # collective stand-in: real inputs for the merge
        if not torch.equal(judges[0].sel, sel_ref):
            raise RuntimeError(f"band-merged modes differ from the whole-frame judge (N={n})")
        t_merge = max(timed(lambda j=j: j.merge_owned(), steps) for j in judges)
        t_select = timed(lambda: judges[0].select(), steps)
        t_emit = max(timed(lambda j=j: j.emit(frames), steps) for j in judges)
        per_rank = max(part) + t_merge + t_select + t_emit
        q = judges[0].q
        # the peer exchange: each owner pulls its slots' rows from every band
        # and pushes the entropies (pcbz_judge_merge_peers_device); here the
        # "peers" are buffers on this GPU, so the pull reads local HBM where
        # a real rank reads (n-1)/n of it over NVLink (reported in bytes)
        peers = [BandJudge((F, H, W), pitch, wl.codes, wl.temporal, False, b, n, exchange="peer")
                 for b in range(n)]
        emulate_band_peer_exchange(peers, [(frames, None)] * n)
        if not all(torch.equal(j.sel, sel_ref) for j in peers):
            raise RuntimeError(f"peer-exchange modes differ from the whole-frame judge (N={n})")
        t_merge_peers = max(timed(lambda j=j: j.merge_peers(), steps) for j in peers)
        t_signal = timed(lambda: (peers[0].signal(2, 1), peers[0].signal(2, 2)), steps)   # already met: launch cost
        print(json.dumps({
            "workload": name, "bands": n, "segments_per_band": judges[0].segments,
            "partial_ms_per_band": part, "merge_owned_ms_max_rank": t_merge, "select_ms": t_select,
            "emit_ms_max_band": t_emit, "per_rank_compute_ms": per_rank,
            "owned_slots_per_rank": q,
            "reduce_scatter_bytes_sent_per_rank": (n - 1) * q * 65536 * 4,
            "all_to_all_bytes_sent_per_rank": (n - 1) * q * judges[0].segments * 512 * 2,
            "all_gather_bytes_per_rank": q * 8,
            "merge_peers_ms_max_rank": t_merge_peers,
            "peer_signal_pair_ms": t_signal,
            "peer_pull_bytes_remote_per_rank": (n - 1) * q * (65536 * 4 + judges[0].segments * 512 * 2),
            "per_rank_compute_ms_peer_exchange": max(part) + t_merge_peers + 2 * t_signal + t_select + t_emit,
            "GBps_raw_excluding_collective": raw / (per_rank * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
