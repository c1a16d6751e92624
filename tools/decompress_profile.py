"""Wall-clock breakdown of decompress_stack on 100 C2 frames: bzip2 decoding
of every payload on the host pool vs the rest (symbol unpacking, inverse
prediction on the GPU).  python tools/decompress_profile.py"""
import bz2
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry,  # noqa: E402
                                   all_intra_specs, compress_stack, decompress_stack)
from paper_2310_09467_b200.codec import read_container  # noqa: E402

wl = bench.WORKLOADS["c2"]
cores = os.cpu_count() or 1
host = bench.make_frames(wl, range(100), cores)
geo = LensletGeometry(15, 15)
stack = FrameStack(tuple(Frame(f, geo) for f in host))
data = compress_stack(stack, CompressOptions(workers=cores, temporal=False, candidates=tuple(all_intra_specs())))
decompress_stack(data, workers=cores)
t0 = time.perf_counter()
back = decompress_stack(data, workers=cores)
t_all = time.perf_counter() - t0
from paper_2310_09467_b200 import pipeline  # noqa: E402
hdr, records, payloads = read_container(data)
t0 = time.perf_counter()
fast = pipeline._decompress_device(hdr, records, payloads)
t_dev = time.perf_counter() - t0
print(f"device path: {'taken' if fast is not None else 'NOT taken'}, {t_dev:.3f} s", flush=True)
jobs = [bytes(p) for ps in payloads for p in ps]
t0 = time.perf_counter()
with ThreadPoolExecutor(cores) as ex:
    out = list(ex.map(bz2.decompress, jobs))
t_bz = time.perf_counter() - t0
t0 = time.perf_counter()
x = bz2.decompress(jobs[0])
t_one = time.perf_counter() - t0
print(f"decompress_stack {t_all:.3f} s; bz2 of {len(jobs)} payloads on {cores} threads {t_bz:.3f} s; "
      f"one payload single-threaded {t_one * 1e3:.1f} ms ({len(x) / t_one / 1e6:.0f} MB/s)")
