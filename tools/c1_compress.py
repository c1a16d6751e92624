import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from workloads.configs import WORKLOADS, make_frames
from paper_2310_09467_b200 import CompressOptions, Frame, FrameStack, LensletGeometry, compress_stack, decompress_stack
vol = make_frames(WORKLOADS['c1'], range(1))
stack = FrameStack((Frame(vol[0], LensletGeometry(15, 15)),))
for coder in ('device', 'host'):
    opts = CompressOptions(workers=os.cpu_count(), coder=coder)
    compress_stack(stack, opts)
    t = time.perf_counter()
    for _ in range(3): data = compress_stack(stack, opts)
    dt = (time.perf_counter() - t) / 3
    decompress_stack(data, workers=os.cpu_count())
    t = time.perf_counter()
    for _ in range(3): back = decompress_stack(data, workers=os.cpu_count())
    dd = (time.perf_counter() - t) / 3
    print(coder, f"compress {dt*1e3:.1f} ms, decompress {dd*1e3:.1f} ms, CR {vol.nbytes/len(data):.3f}", np.array_equal(back.to_array(), vol))
