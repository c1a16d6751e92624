"""bench.py's multi-GPU plumbing on CPU: the `--gpus N` launch plan (one
rank per GPU under torch.distributed.run), the refusal when fewer GPUs are
visible, the rank reductions (max-over-ranks timing, summed bytes) over a
2-rank gloo group, and the frame-shard split with its one-frame halo."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from workloads.configs import ALL26, Workload, make_frames

SMALL = Workload("t", "test series", 7, 48, 64, 15, ALL26, True, True)


def test_launch_plan_two_ranks():
    args = bench.parse_args(["--gpus", "2", "--steps", "4", "--warmup", "3"])
    cmd, err = bench.launch_plan(args, ["--gpus", "2", "--steps", "4", "--warmup", "3"], 2, 29555)
    assert err is None
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-6:] == ["--gpus", "2", "--steps", "4", "--warmup", "3"]
    assert cmd[-7].endswith("bench.py")


def test_launch_plan_refuses_missing_gpus():
    args = bench.parse_args(["--gpus", "8"])
    cmd, err = bench.launch_plan(args, ["--gpus", "8"], 1, 29555)
    assert cmd is None and "8 visible GPUs" in err


def test_main_exits_nonzero_without_gpus(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 1)
    assert bench.main(["--gpus", "2", "--no-cpu-baseline", "--no-pipeline"]) == 2


def test_main_checks_world_size(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--gpus", "4"]) == 2


def test_configs_identical_on_both_arms():
    wl = bench.WORKLOADS["c2"]
    for world in (1, 2, 8):
        assert bench.config(wl, world, "frames") == bench.config(wl, world, "frames")
        assert bench.config(wl, world)["parallelism"] == ("single GPU" if world == 1 else f"replicas x{world} (no collective)")


def _ranks_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = bench.Ranks(world, torch.device("cpu"))
        r.barrier()
        out[rank] = (r.max(float(rank + 1) * 1.5), r.sum(float(100 * (rank + 1))))
    finally:
        dist.destroy_process_group()


def test_rank_reductions_gloo():
    port = bench._free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_ranks_worker, args=(2, port, out), nprocs=2, join=True)
        assert dict(out) == {0: (3.0, 300.0), 1: (3.0, 300.0)}


@pytest.mark.parametrize("world", [1, 2, 3])
def test_rank_frames_shards_cover_series(world):
    whole = make_frames(SMALL, range(SMALL.frames))
    seen = []
    for rank in range(world):
        fr, halo, first = bench.rank_frames(SMALL, world, rank, 2)
        assert np.array_equal(fr, whole[first:first + fr.shape[0]])
        if first == 0:
            assert halo is None
        else:
            assert np.array_equal(halo, whole[first - 1])
        seen.extend(range(first, first + fr.shape[0]))
    assert seen == list(range(SMALL.frames))


def test_reference_arm_other_ranks_exit_without_work(monkeypatch, capsys):
    """Under torchrun the reference arm runs on rank 0 only; other ranks
    print nothing and exit 0."""
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(bench, "make_frames", lambda *a, **k: (_ for _ in ()).throw(AssertionError("worked")))
    assert bench.main(["--impl", "reference", "--gpus", "2"]) == 0
    assert capsys.readouterr().out == ""
