"""GPU bzip2 back end vs the host coder on the pipeline's real input: the
residual streams of C2 frames cut into 4 MiB PCBZ blocks (one
bz2.compress(chunk, 9) per block, reference blocks.py:73-81).

    python tools/bench_bzip2.py [nframes]
"""
import bz2
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200 import LensletGeometry, pipeline  # noqa: E402
from paper_2310_09467_b200.codec import bz2_blocks_device, split_blocks  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    cores = os.cpu_count() or 1
    wl = bench.WORKLOADS["c2"]
    vol = bench.make_frames(wl, range(n), cores)
    _, sel, streams = pipeline.judge_volume(vol, LensletGeometry(15, 15), list(range(13)), False)
    chunks = [bytes(b) for s in streams for b in split_blocks(s, 4 << 20)]
    raw = sum(len(c) for c in chunks)
    bz2_blocks_device(chunks[:2])                       # warm-up (context, buffers)
    t0 = time.perf_counter()
    gpu = bz2_blocks_device(chunks)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        host = list(ex.map(lambda c: bz2.compress(c, 9), chunks))
    t_host = time.perf_counter() - t0
    same = all(a == b for a, b in zip(gpu, host))
    print(json.dumps({"frames": n, "jobs": len(chunks), "input_bytes": raw,
                      "compressed_bytes": sum(len(c) for c in host), "identical": same,
                      "gpu_s": t_gpu, "gpu_GBps": raw / t_gpu / 1e9,
                      "host_s": t_host, "host_GBps": raw / t_host / 1e9, "host_threads": cores}), flush=True)


if __name__ == "__main__":
    main()
