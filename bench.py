"""Benchmark of the entropy-judgement stage (BASELINE.json metric:
"entropy-judge GB/s raw uint16 LFM at 1/2/4/8 B200; % HBM peak; CR parity").

Workload (BASELINE.json configs[1]): 100 independent
synthetic 2048x2048 uint16 bead frames, pitch 15x15, three SNR levels
(34 high: amp 20000 sigma 0 photon 0.05; 33 mid: amp 3000 sigma 100 photon
0.05; 33 low: amp 3000 sigma 500 photon 0.01), seeds 0..99, generated
bit-identically to the reference's synth.generate; 13 intra candidates
(independent frames, temporal off).

One step = judge + emission of the whole batch: per-candidate approximate-BWT
pair histograms, fp64 entropies, argmin, selected big-endian residual streams.
`value` = raw frame bytes (2*H*W per frame, all ranks) / step time, frames
resident in HBM.  `e2e` = same metric through the public host API with pinned
host buffers (H2D of frames + D2H of streams and modes inside the timed
region).  Inputs (839 MB) exceed the 126 MB L2, so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

H = W = 2048
PITCH = 15
N_FRAMES = 100
CODES = list(range(13))
METRIC = "entropy-judge GB/s raw uint16 LFM at 1/2/4/8 B200; % HBM peak; CR parity"
SNR_LEVELS = [  # (count, amplitude, sigma, photon) -- SURVEY.md §8(d) C2
    (34, 20000.0, 0.0, 0.05),
    (33, 3000.0, 100.0, 0.05),
    (33, 3000.0, 500.0, 0.01),
]


def frame_params():
    from paper_2310_09467_b200.lfm_synth import SynthParams
    out, seed = [], 0
    for count, amp, sigma, photon in SNR_LEVELS:
        for _ in range(count):
            out.append(SynthParams(W, H, PITCH, PITCH, mode="beads", signal_amplitude=amp,
                                   noise_sigma=sigma, photon_scale=photon, frames=1, seed=seed))
            seed += 1
    return out


def _gen_one(p):
    from paper_2310_09467_b200.lfm_synth import generate_array
    return generate_array(p)[0]


def make_frames(n: int, workers: int) -> np.ndarray:
    params = frame_params()[:n]
    vol = np.empty((n, H, W), np.uint16)
    with ProcessPoolExecutor(max(1, workers)) as ex:
        for i, fr in enumerate(ex.map(_gen_one, params, chunksize=2)):
            vol[i] = fr
    return vol


def config(extra=None):
    c = {"workload": "C2: 100 independent 2048x2048 uint16 bead frames, pitch 15x15, 3 SNR levels, "
                     "13 intra candidates, judge + emission",
         "frames_per_gpu": N_FRAMES, "height": H, "width": W, "pitch": [PITCH, PITCH],
         "candidates": len(CODES), "l2_policy": "inputs (839 MB/GPU) larger than L2 (126 MB), no flush"}
    if extra:
        c.update(extra)
    return c


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def cpu_reference_sample(vol: np.ndarray, nthreads: int):
    """Time the CPU port of the reference path (oracle, C, pthreads) on a
    bounded sample; returns (GB/s raw, seconds, frames)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    oracle.select_batch(vol[:1, :64, :64], None, CODES, PITCH, PITCH, nthreads=1)   # load/warm
    t0 = time.perf_counter()
    oracle.select_batch(vol, None, CODES, PITCH, PITCH, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return vol.shape[0] * 2 * H * W / dt / 1e9, dt, vol.shape[0]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    sample_frames = int(os.environ.get("PCBZ_REF_SAMPLE_FRAMES", "16"))
    vol = make_frames(sample_frames, cores)
    for _ in range(args.warmup):
        cpu_reference_sample(vol[:max(1, sample_frames // 4)], cores)
    times = []
    for _ in range(args.steps):
        _, dt, _ = cpu_reference_sample(vol, cores)
        times.append(dt)
    t = statistics.mean(times)
    v = sample_frames * 2 * H * W / t / 1e9
    sample = f"{sample_frames} of the 100 C2 frames per step, judge (13 candidates) + emission"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": config({"sample_frames_per_step": sample_frames}),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2310_09467_b200 import LensletGeometry, pipeline
    from paper_2310_09467_b200.device import DeviceJudge, collect_timing, set_profiling

    cores = os.cpu_count() or 1
    host = make_frames(N_FRAMES, max(1, cores // world))
    pinned = torch.empty((N_FRAMES, H, W), dtype=torch.uint16).pin_memory()
    pinned.numpy()[...] = host
    frames = pinned.to(dev)
    judge = DeviceJudge((N_FRAMES, H, W), (PITCH, PITCH), CODES, temporal=False, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region ----------------------------------------
    for _ in range(args.warmup):
        judge(frames)
    barrier()
    set_profiling(True)
    collect_timing()
    with ClockSampler(local) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            judge(frames)
        e1.record(stream)
        barrier()
    set_profiling(False)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    hist_ms_sum, judge_ms_sum, launches = collect_timing()
    hist_ms = max_over_ranks(hist_ms_sum / args.steps)
    raw_bytes = N_FRAMES * 2 * H * W
    value = world * raw_bytes / (ms * 1e-3) / 1e9

    # ---- end to end through the public host API (pinned buffers) -------------
    geo = LensletGeometry(PITCH, PITCH)
    vol_np = pinned.numpy()
    ent_h = torch.empty((N_FRAMES, len(CODES)), dtype=torch.float64).pin_memory().numpy()
    sel_h = torch.empty(N_FRAMES, dtype=torch.uint8).pin_memory().numpy()
    stream_h = torch.empty((N_FRAMES, 2 * H * W), dtype=torch.uint8).pin_memory().numpy()
    out = (ent_h, sel_h, stream_h)
    pipeline.judge_volume(vol_np, geo, CODES, False, out=out)
    e2e_steps = max(1, min(args.steps, 5))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pipeline.judge_volume(vol_np, geo, CODES, False, out=out)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_value = world * raw_bytes / e2e_s / 1e9
    # parity spot check of the e2e output against the device-resident run
    if not np.array_equal(sel_h, judge.sel.cpu().numpy()):
        raise RuntimeError("e2e and device-resident selections differ")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_kind = measured_peak_hbm()
    alg_bytes_hist = raw_bytes            # the histogram kernel reads every frame once
    achieved = alg_bytes_hist / (hist_ms * 1e-3) / 1e9
    stage_bytes = 2 * raw_bytes           # stage: read frames + write streams
    traffic = None
    tf = ROOT / "profiles" / "latest_hist_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("bytes_per_launch")
    res = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16", "data": "synthetic (reference synth.generate, bit-identical)",
        "config": config({"parallelism": f"frames x{world} (replicas, no collective)" if world > 1 else "single GPU"}),
        "roofline": {"bound": "hbm", "kernel": "judge_hist_kernel", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_kind": peak_kind, "hist_kernel_ms": hist_ms,
                     "algorithmic_bytes_per_launch": alg_bytes_hist,
                     "stage_frac": (stage_bytes / (ms * 1e-3) / 1e9) / peak,
                     "events_per_s": N_FRAMES * len(CODES) * (2 * H * W) / (hist_ms * 1e-3)},
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": raw_bytes,
                "d2h_bytes_per_step": stream_h.nbytes + ent_h.nbytes + sel_h.nbytes,
                "api": "paper_2310_09467_b200.pipeline.judge_volume (pcbz_judge_host)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        sample = int(os.environ.get("PCBZ_CPU_SAMPLE_FRAMES", "16"))
        v, dt, nf = cpu_reference_sample(host[:sample], cores)
        res["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                               "sample": f"{nf} C2 frames, judge (13 candidates) + emission, {dt:.2f} s wall"}
    print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
