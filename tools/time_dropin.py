"""Per-frame drop-in path: the reference's compress_stack_detailed with its
select_predictor routed to the B200 (install(level="api")) vs unpatched, on
C2 frames; plus this package's criterion.select_predictor per frame
(pageable numpy, the reference signature)."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pcbz_numba_cache")

import numpy as np  # noqa: E402

from paper_2310_09467_b200 import Frame, LensletGeometry, criterion  # noqa: E402
from workloads.configs import WORKLOADS, make_frames  # noqa: E402

vol = make_frames(WORKLOADS["c2"], range(8), os.cpu_count() or 1)
geo = LensletGeometry(15, 15)
out = {}
fr = [Frame(v, geo) for v in vol]
criterion.select_predictor(fr[0])
t0 = time.perf_counter()
for f in fr:
    criterion.select_predictor(f)
out["select_predictor_ms_per_frame"] = (time.perf_counter() - t0) / len(fr) * 1e3
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import pcbz  # noqa: E402
from pcbz import _kernels as rk  # noqa: E402
rk.warm_up()
stack = pcbz.FrameStack(tuple(pcbz.Frame(v, pcbz.LensletGeometry(15, 15)) for v in vol))
opts = pcbz.CompressOptions(workers=os.cpu_count(), temporal=False)
r0 = pcbz.compress_stack_detailed(stack, opts)
out["reference_numba"] = {"select_s_per_frame": r0.select_seconds / len(vol), "encode_s_per_frame": r0.encode_seconds / len(vol)}
import paper_2310_09467_b200 as b200  # noqa: E402
b200.install(pcbz, level="api")
pcbz.compress_stack_detailed(stack, opts)
r1 = pcbz.compress_stack_detailed(stack, opts)
out["reference_installed_api"] = {"select_s_per_frame": r1.select_seconds / len(vol), "encode_s_per_frame": r1.encode_seconds / len(vol),
                                  "same_bytes": r1.data == r0.data}
b200.install(pcbz, level="pipeline")
pcbz.compress_stack_detailed(stack, opts)
t0 = time.perf_counter()
r2 = pcbz.compress_stack_detailed(stack, opts)
wall = time.perf_counter() - t0
out["reference_installed_pipeline"] = {"select_s_per_frame": r2.select_seconds / len(vol),
                                       "encode_s_per_frame": r2.encode_seconds / len(vol),
                                       "wall_s_per_frame": wall / len(vol), "same_bytes": r2.data == r0.data}
out["reference_unpatched_wall_s_per_frame"] = (r0.select_seconds + r0.encode_seconds) / len(vol)
print(json.dumps(out))
