"""Per-rank cost of frame sharding measured on
ONE GPU: for N ranks, rank r's shard of the series (contiguous frames plus
the one-frame halo, bench.rank_frames / shard.plan_frame_shards) is judged
alone -- what rank r runs, with no collective on the data path -- and the
slowest rank's device time gives the projected strong-scaling step.

    python tools/shard_projection.py [c3|c4] [steps]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2310_09467_b200.device import DeviceJudge  # noqa: E402
from paper_2310_09467_b200.shard import plan_frame_shards  # noqa: E402
from workloads.configs import WORKLOADS, make_frames  # noqa: E402


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
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = WORKLOADS[name]
    F, H, W = wl.frames, wl.height, wl.width
    vol = make_frames(wl, range(F), os.cpu_count() or 1)
    frames = torch.from_numpy(vol).cuda()
    raw = F * 2 * H * W
    t1 = None
    for n in (1, 2, 4, 8):
        per_rank = []
        sels = []
        for sh in plan_frame_shards(F, n, wl.temporal):
            fr = frames[sh.begin:sh.end].contiguous()
            halo = frames[sh.halo].contiguous() if sh.halo is not None else None
            j = DeviceJudge(tuple(fr.shape), (wl.pitch, wl.pitch), wl.codes, temporal=wl.temporal)
            per_rank.append(timed(lambda: j(fr, halo), steps))
            sels.append(j.sel.clone())
        sel = torch.cat(sels)
        if t1 is None:
            t1, sel1 = max(per_rank), sel
        elif not torch.equal(sel, sel1):
            raise RuntimeError(f"sharded selections differ from the one-rank judge (N={n})")
        ms = max(per_rank)
        print(json.dumps({"workload": name, "ranks": n, "frames_per_rank": [sh.count for sh in plan_frame_shards(F, n, wl.temporal)],
                          "rank_ms": per_rank, "step_ms_max_over_ranks": ms,
                          "projected_GBps": raw / (ms * 1e-3) / 1e9, "speedup_vs_1": t1 / ms,
                          "efficiency": t1 / ms / n}), flush=True)


if __name__ == "__main__":
    main()
