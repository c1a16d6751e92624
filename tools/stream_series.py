"""Config C3 end to end: a long
smooth_lenslet time series (default 1000 frames of 2048^2, 8.39 GB raw)
generated on the fly (reference synth RNG keys, lfm_synth), compressed by
pipeline.compress_stream -- device judge + emission in chunks, bzip2 on all
host threads -- into a seekable byte-counting sink.  Memory stays bounded
(peak RSS reported); the whole series is never materialised.

    python tools/stream_series.py [nframes] [chunk_frames]
"""
import io
import json
import multiprocessing as mp
import os
import resource
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import workloads.configs as wc  # noqa: E402
import workloads.configs as wc  # noqa: E402
from paper_2310_09467_b200 import CompressOptions, LensletGeometry  # noqa: E402
from paper_2310_09467_b200.pipeline import compress_stream  # noqa: E402


class CountingSink(io.RawIOBase):
    """Seekable sink that keeps no data: position bookkeeping only."""

    def __init__(self):
        self.pos = self.size = 0

    def writable(self):
        return True

    def seekable(self):
        return True

    def write(self, b):
        n = len(b)
        self.pos += n
        self.size = max(self.size, self.pos)
        return n

    def tell(self):
        return self.pos

    def seek(self, off, whence=0):
        self.pos = off if whence == 0 else (self.pos + off if whence == 1 else self.size + off)
        return self.pos


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    wl = bench.Workload("c3", "C3", n, 2048, 2048, 15, tuple(bench.ALL26), True, True)
    from workloads.lfm_synth import scene
    p = bench.series_params(wl)
    wc._SERIES["base"], wc._SERIES["params"] = scene(p), p   # inherited by forked workers
    cores = os.cpu_count() or 1
    gen_procs = max(1, cores // 2)
    ctx = mp.get_context("fork")
    sink = CountingSink()
    t0 = time.perf_counter()
    with ctx.Pool(gen_procs) as pool:
        frames = pool.imap(wc._gen_series_frame, range(n), chunksize=2)
        res = compress_stream(frames, LensletGeometry(15, 15), sink,
                              CompressOptions(workers=cores), nframes=n, chunk_frames=chunk)
    dt = time.perf_counter() - t0
    raw = n * 2 * 2048 * 2048
    print(json.dumps({
        "workload": f"C3: {n}-frame 2048x2048 smooth_lenslet series, pitch 15, drift 1, temporal on",
        "frames": res.frames, "raw_bytes": raw, "container_bytes": res.container_bytes,
        "compression_ratio": raw / res.container_bytes, "wall_s": dt, "GBps_raw_e2e": raw / dt / 1e9,
        "device_judge_s": res.select_seconds, "host_threads": cores, "generator_processes": gen_procs,
        "peak_rss_MB": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024,
        "note": "e2e includes on-the-fly synthesis (generator processes share the host cores with bzip2)"}),
        flush=True)


if __name__ == "__main__":
    main()
