"""Frame sharding (multi-GPU path) on CPU: world-size-2 gloo process group,
the CPU oracle standing in for each rank's device judge.  The assembled
container must equal the single-process reference restatement."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import sha
from paper_2310_09467_b200.core import LensletGeometry
from paper_2310_09467_b200.lfm_synth import SynthParams, generate_array
from paper_2310_09467_b200.shard import compress_sharded, plan_frame_shards


def oracle_judge(frames, halo, geo, codes, temporal):
    """Per-rank judge: the oracle restatement of select_predictor + emission."""
    F = frames.shape[0]
    ent = np.full((F, len(codes)), np.nan)
    sel = np.zeros(F, np.uint8)
    streams = []
    prev = halo
    for f in range(F):
        cands = [c for c in codes if (prev is not None and temporal) or not c & 0x80]
        entries, best, _ = oracle.select_predictor(frames[f], prev if temporal else None, cands,
                                                   geo.pitch_x, geo.pitch_y)
        for c, e in entries:
            ent[f, codes.index(c)] = e
        sel[f] = best
        streams.append(np.frombuffer(oracle.emit_stream(frames[f], prev, best, geo.pitch_x,
                                                        geo.pitch_y), np.uint8))
        prev = frames[f]
    return ent, sel, np.stack(streams)


def test_plan_balanced_and_halo():
    plans = plan_frame_shards(10, 4)
    assert [(p.begin, p.end) for p in plans] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert [p.halo for p in plans] == [None, 2, 5, 7]
    assert [p.halo for p in plan_frame_shards(10, 4, temporal=False)] == [None] * 4
    assert sum(p.count for p in plan_frame_shards(3, 8)) == 3
    with pytest.raises(ValueError):
        plan_frame_shards(0, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, vol, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    codes = list(range(13)) + [0x80 | i for i in range(13)]
    data = compress_sharded(vol, LensletGeometry(6, 5), codes, True, 4 * 1024 * 1024, rank, world,
                            judge_fn=oracle_judge)
    if rank == 0:
        out.put(data)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_container_equals_single_process():
    vol = generate_array(SynthParams(40, 33, 6, 5, mode="smooth_lenslet", noise_sigma=30.0,
                                     photon_scale=0.05, frames=5, drift=0.5, seed=7))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, vol, q)) for r in range(2)]
    for p in procs:
        p.start()
    data = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want, _ = oracle.compress_stack(vol, 6, 5)
    assert sha(data) == sha(want)
