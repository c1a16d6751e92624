import os, sys, ctypes, numpy as np
sys.path.insert(0, '/root/repo')
import torch
from paper_2310_09467_b200 import _lib
from paper_2310_09467_b200.device import DeviceJudge
from workloads.configs import WORKLOADS, make_frames
wl = WORKLOADS['c2']
vol = make_frames(wl, range(100), os.cpu_count())
fr = torch.from_numpy(vol).cuda()
j = DeviceJudge(vol.shape, (15, 15), wl.codes, temporal=False)
j(fr); torch.cuda.synchronize()
lib = _lib.load(); lib.pcbz_set_item_trace(1); j(fr); torch.cuda.synchronize()
W = int(os.environ.get('PCBZ_TRACE_WORDS', '5'))
buf = np.zeros(W * 4096, np.uint64); seg = ctypes.c_int()
n = lib.pcbz_item_trace(buf.ctypes.data, 4096, ctypes.byref(seg)); lib.pcbz_set_item_trace(0)
r = buf[:W * n].reshape(n, W).astype(np.int64)
t0 = r[:, 0] & ((1 << 48) - 1); t0 = t0 + ((r[:, 2] >> 48) << 48); t0 = np.where(t0 > r[:, 2], t0 - (1 << 48), t0)
runs, claim, stitch, end = r[:, 1], r[:, 3], r[:, 4], r[:, 2]
print({"items": int(n), "runs_us": float(((runs - t0) / 1e3).mean()), "claim_sweep_us": float(((claim - runs) / 1e3).mean()),
       "stitch_us": float(((stitch - claim) / 1e3).mean()), "seams_entropy_us": float(((end - stitch) / 1e3).mean())})
if W >= 9:
    b, sc, tr, lv = r[:, 5], r[:, 6], r[:, 7], r[:, 8]
    print({"seams_spill_bitmap_occ_us": float(((b - stitch) / 1e3).mean()), "scan_us": float(((sc - b) / 1e3).mean()),
           "tree_us": float(((tr - sc) / 1e3).mean()), "leaves_us": float(((lv - tr) / 1e3).mean()),
           "fold_us": float(((end - lv) / 1e3).mean())})
