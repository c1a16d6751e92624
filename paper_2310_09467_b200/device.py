"""Device-resident batched judge on torch CUDA tensors (the fast path behind
pcbz_judge_device).  torch is plumbing here: device memory and the stream the
kernels are enqueued on; all compute is libpcbz_b200.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class DeviceJudge:
    """Judge + emit for [F, H, W] uint16 frames already in device memory.

    Reusable: the workspace is sized once per (F, H, W, k, want_hist) shape.
    Outputs are device tensors: ent [F, k] float64 (NaN = not scored),
    sel [F] uint8, stream [F, 2*H*W] uint8 (big-endian residual bytes).
    """

    def __init__(self, frames_shape, pitch, codes, temporal: bool, want_stream: bool = True,
                 want_hist: bool = False, device=None):
        import torch

        self.torch = torch
        F, H, W = frames_shape
        self.F, self.H, self.W = F, H, W
        self.px, self.py = pitch
        self.codes = np.array(sorted(int(c) for c in codes), np.uint8)
        self.k = int(self.codes.size)
        self.temporal = 1 if temporal else 0
        self.device = torch.device(device or "cuda")
        lib = _lib.load()
        ws = lib.pcbz_judge_workspace_size(F, H, W, self.k, 1 if want_hist else 0)
        if ws == 0:
            raise ValueError("invalid judge shape")
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        self.ent = torch.empty((F, self.k), dtype=torch.float64, device=self.device)
        self.sel = torch.empty(F, dtype=torch.uint8, device=self.device)
        self.stream = (torch.empty((F, 2 * H * W), dtype=torch.uint8, device=self.device)
                       if want_stream else None)
        self.hist = (torch.empty((F, self.k, 65536), dtype=torch.int32, device=self.device)
                     if want_hist else None)

    def __call__(self, frames, halo=None, stream=None):
        """Enqueue on `stream` (default: torch's current stream); no sync."""
        t = self.torch
        assert frames.dtype == t.uint16 and frames.is_contiguous() and tuple(frames.shape) == (self.F, self.H, self.W)
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        rc = _lib.load().pcbz_judge_device(
            frames.data_ptr(), halo.data_ptr() if halo is not None else None, self.F, self.H,
            self.W, self.px, self.py, self.codes.ctypes.data, self.k, self.temporal,
            self.ent.data_ptr(), self.sel.data_ptr(),
            self.stream.data_ptr() if self.stream is not None else None,
            self.hist.data_ptr() if self.hist is not None else None,
            self.workspace.data_ptr(), self.workspace.numel(), ctypes.c_void_p(st.cuda_stream))
        _lib.check(rc)
        return self.ent, self.sel, self.stream


def set_profiling(on: bool) -> None:
    _lib.load().pcbz_set_profiling(1 if on else 0)


def collect_timing():
    """(sum of histogram-kernel ms, sum of whole-judge ms, kernels launched)
    since the previous call (see pcbz_last_timing)."""
    h = ctypes.c_float()
    t = ctypes.c_float()
    n = ctypes.c_int()
    _lib.check(_lib.load().pcbz_last_timing(ctypes.byref(h), ctypes.byref(t), ctypes.byref(n)))
    return h.value, t.value, n.value
