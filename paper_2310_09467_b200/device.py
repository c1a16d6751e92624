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
        with torch.cuda.device(self.device):
            _lib.ensure_entropy_terms(2 * H * W - 1)
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


class BandJudge:
    """One rank's share of a judge whose streams are split into `nbands`
    within-frame pixel bands (pcbz_judge_band_device / _merge_device /
    _emit_band_device; include/pcbz_b200.h).  Frames and halo are resident on
    every rank; each rank scores its band, the partial histograms are summed
    and the segment summaries gathered across ranks (shard.band_collective),
    then every rank finishes the identical entropies / modes and emits its
    band of every stream.

    Buffers: hist [F*k, 65536] int32 (partial, then summed in place),
    summary [F*k*S*512] int16 (this band), summaries [nbands, F*k*S*512]
    (gathered, band order), ent [F, k], sel [F], stream [F, 2*(end-begin)].
    """

    def __init__(self, frames_shape, pitch, codes, temporal: bool, has_halo: bool, band: int,
                 nbands: int, want_stream: bool = True, device=None):
        import torch

        self.torch = torch
        F, H, W = frames_shape
        self.F, self.H, self.W = F, H, W
        self.px, self.py = pitch
        self.codes = np.array(sorted(int(c) for c in codes), np.uint8)
        self.k = int(self.codes.size)
        self.temporal = 1 if temporal else 0
        self.has_halo = 1 if has_halo else 0
        self.band, self.nbands = int(band), int(nbands)
        self.device = torch.device(device or "cuda")
        lib = _lib.load()
        with torch.cuda.device(self.device):
            _lib.ensure_entropy_terms(2 * H * W - 1)
        S, sb, ws = ctypes.c_int(), ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(lib.pcbz_band_layout(F, H, W, self.px, self.py, self.codes.ctypes.data, self.k,
                                        self.temporal, self.has_halo, self.nbands, ctypes.byref(S),
                                        ctypes.byref(sb), ctypes.byref(ws)))
        self.segments = S.value
        b0, b1 = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.pcbz_band_range(H, W, self.nbands, self.band, ctypes.byref(b0), ctypes.byref(b1)))
        self.pix_begin, self.pix_end = b0.value, b1.value
        dev = self.device
        self.workspace = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=dev)
        self.hist = torch.empty((F * self.k, 65536), dtype=torch.int32, device=dev)
        self.summary = torch.empty(sb.value // 2, dtype=torch.int16, device=dev)
        self.summaries = torch.empty((self.nbands, sb.value // 2), dtype=torch.int16, device=dev)
        self.ent = torch.empty((F, self.k), dtype=torch.float64, device=dev)
        self.sel = torch.empty(F, dtype=torch.uint8, device=dev)
        self.stream = (torch.empty((F, 2 * (self.pix_end - self.pix_begin)), dtype=torch.uint8, device=dev)
                       if want_stream else None)

    def _st(self, stream):
        t = self.torch
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        return ctypes.c_void_p(st.cuda_stream)

    def _check_frames(self, frames, halo):
        t = self.torch
        assert frames.dtype == t.uint16 and frames.is_contiguous() and tuple(frames.shape) == (self.F, self.H, self.W)
        if (halo is not None) != bool(self.has_halo):
            raise ValueError("halo presence differs from the layout this BandJudge was built for")

    def partial(self, frames, halo=None, stream=None):
        """This band's partial histograms and segment summaries (enqueued)."""
        self._check_frames(frames, halo)
        rc = _lib.load().pcbz_judge_band_device(
            frames.data_ptr(), halo.data_ptr() if halo is not None else None, self.F, self.H,
            self.W, self.px, self.py, self.codes.ctypes.data, self.k, self.temporal, self.band,
            self.nbands, self.hist.data_ptr(), self.summary.data_ptr(), self.workspace.data_ptr(),
            self.workspace.numel(), self._st(stream))
        _lib.check(rc)
        return self.hist, self.summary

    def merge(self, stream=None):
        """Entropies and modes from the SUMMED hist and GATHERED summaries."""
        rc = _lib.load().pcbz_judge_merge_device(
            self.F, self.H, self.W, self.px, self.py, self.codes.ctypes.data, self.k, self.temporal,
            self.has_halo, self.nbands, self.hist.data_ptr(), self.summaries.data_ptr(),
            self.ent.data_ptr(), self.sel.data_ptr(), self._st(stream))
        _lib.check(rc)
        return self.ent, self.sel

    def emit(self, frames, halo=None, stream=None):
        """This band's residual bytes of every frame under self.sel."""
        self._check_frames(frames, halo)
        if self.stream is None:
            return None
        rc = _lib.load().pcbz_emit_band_device(
            frames.data_ptr(), halo.data_ptr() if halo is not None else None, self.F, self.H,
            self.W, self.px, self.py, self.sel.data_ptr(), self.band, self.nbands,
            self.stream.data_ptr(), self._st(stream))
        _lib.check(rc)
        return self.stream

    def __call__(self, frames, halo=None, group=None, stream=None):
        """partial -> all-reduce / all-gather over `group` -> merge -> emit."""
        import contextlib

        from .shard import band_collective

        # the collectives order against torch's current stream: run the whole
        # partial -> collective -> merge -> emit sequence on `stream` as current
        ctx = self.torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            return band_collective(lambda: self.partial(frames, halo, stream), self.summaries,
                                   lambda: self.merge(stream), lambda: self.emit(frames, halo, stream),
                                   self.nbands, group)


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
