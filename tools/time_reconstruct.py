"""Wall-clock of the inverse prediction entry points on a C2-sized frame
(per-frame `_kernels.reconstruct_image`, host buffers, i.e. what install()
routes the reference's decompress to) and a 100-frame batch
(`pcbz_reconstruct_host`), against the reference's numba kernel when
baseline/_ref is importable."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2310_09467_b200 import _kernels, _lib  # noqa: E402
from workloads.configs import WORKLOADS, make_frames  # noqa: E402

vol = make_frames(WORKLOADS["c2"], range(8), os.cpu_count() or 1)
out = {}
for cid in (0, 1, 5, 12):
    res = oracle.residual_image(vol[0], cid, 15, 15)
    _kernels.reconstruct_image(res, cid, 15, 15)
    t0 = time.perf_counter()
    for _ in range(5):
        back = _kernels.reconstruct_image(res, cid, 15, 15)
    out[f"per_frame_id{cid}_ms"] = (time.perf_counter() - t0) / 5 * 1e3
    assert np.array_equal(back, vol[0])
F = 100
big = np.concatenate([vol] * (F // 8 + 1))[:F]
sel = np.array([12 | (0x80 if f % 2 else 0) for f in range(F)], np.uint8)
sel[0] = 12
res = np.stack([oracle.residual_image(oracle.temporal_delta(big[f], big[f - 1]) if sel[f] & 0x80 else big[f],
                                      12, 15, 15) for f in range(F)])
o = np.empty_like(big)
lib = _lib.load()
for it in range(2):
    t0 = time.perf_counter()
    _lib.check(lib.pcbz_reconstruct_host(_lib.ptr(res), None, F, 2048, 2048, 15, 15, _lib.ptr(sel), _lib.ptr(o)))
    dt = time.perf_counter() - t0
out["batch100_id12_temporal_s"] = dt
assert np.array_equal(o, big)
try:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pcbz_numba_cache")
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    from pcbz import _kernels as rk
    rk.warm_up()
    for cid in (1, 12):
        r = oracle.residual_image(vol[0], cid, 15, 15)
        t0 = time.perf_counter()
        rk.reconstruct_image(r, cid, 15, 15)
        out[f"numba_per_frame_id{cid}_ms"] = (time.perf_counter() - t0) * 1e3
except Exception as e:  # noqa: BLE001
    out["numba"] = repr(e)
print(json.dumps(out))
