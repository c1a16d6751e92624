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
    within-frame pixel bands (pcbz_judge_band_device / _merge_slots_device /
    _select_device / _emit_band_device; include/pcbz_b200.h).  Frames and
    halo are resident on every rank; each rank scores its band, the partial
    histograms are reduce-scattered and the segment summaries exchanged
    all-to-all so that rank r finishes slots [r*q, (r+1)*q) only, the
    entropies are all-gathered and every rank takes the same argmin and
    emits its band of every stream (shard.band_collective).

    Buffers (shard.BandBuffers): hist / summary (this band's partials),
    hist_owned / summ_owned / ent_owned (this rank's slots), ent_all; ent
    [F, k] is a view of ent_all, sel [F], stream [F, 2*(end-begin)].
    """

    def __init__(self, frames_shape, pitch, codes, temporal: bool, has_halo: bool, band: int,
                 nbands: int, want_stream: bool = True, device=None, exchange: str = "nccl",
                 group=None):
        """exchange "nccl": reduce-scatter / all-to-all / all-gather through
        torch.distributed (shard.band_collective); "peer": the exchange
        inside the merge kernel over peer memory (shard.band_peer_exchange)
        -- with a process group the exchanged buffers are allocated in
        symmetric memory and mapped from every rank (NVLink), without one
        the caller wires the peers (attach_peers; one-GPU emulation)."""
        import torch

        from .shard import BandBuffers

        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', got {exchange!r}")
        self.exchange = exchange
        self._epoch = 0
        self._peer_arrays = None

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
        self.nslots = F * self.k
        self.workspace = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=dev)
        shared, symm = None, None
        if exchange == "peer" and group is not None:
            import torch.distributed._symmetric_memory as symm
            shared = lambda shape, dtype: symm.empty(*shape, dtype=dtype, device=dev)  # noqa: E731
        self.buf = BandBuffers.allocate(self.nslots, self.nbands, self.segments * 512, dev, shared)
        # barrier flags of the peer exchange: entry r = last epoch rank r arrived at
        self.flags = (shared((self.nbands,), torch.int32) if shared else
                      torch.empty(self.nbands, dtype=torch.int32, device=dev))
        self.flags.zero_()
        if symm is not None:
            torch.cuda.synchronize(dev)
            handles = [symm.rendezvous(t, group) for t in
                       (self.buf.hist, self.buf.summary, self.buf.ent_all, self.flags)]
            self._set_peer_arrays(*[list(h.buffer_ptrs) for h in handles])
        self.q = self.buf.owned
        self.slot_begin = self.band * self.q
        self.ent = self.buf.ent_all[:self.nslots].view(F, self.k)
        self.sel = torch.empty(F, dtype=torch.uint8, device=dev)
        self.stream = (torch.empty((F, 2 * (self.pix_end - self.pix_begin)), dtype=torch.uint8, device=dev)
                       if want_stream else None)

    @property
    def hist(self):
        return self.buf.hist

    @property
    def summary(self):
        return self.buf.summary

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
            self.nbands, self.buf.hist.data_ptr(), self.buf.summary.data_ptr(), self.workspace.data_ptr(),
            self.workspace.numel(), self._st(stream))
        _lib.check(rc)
        return self.buf.hist, self.buf.summary

    def merge_owned(self, stream=None):
        """Entropies of this rank's slots from buf.hist_owned / buf.summ_owned."""
        rc = _lib.load().pcbz_judge_merge_slots_device(
            self.F, self.H, self.W, self.px, self.py, self.codes.ctypes.data, self.k, self.temporal,
            self.has_halo, self.nbands, self.slot_begin, self.q, self.buf.hist_owned.data_ptr(),
            self.buf.summ_owned.data_ptr(), self.buf.ent_owned.data_ptr(), self._st(stream))
        _lib.check(rc)
        return self.buf.ent_owned

    # ---- peer exchange (shard.band_peer_exchange) ------------------------------
    def _set_peer_arrays(self, hist, summ, ent, flags):
        t = self.torch
        for name, ptrs in (("hist", hist), ("summaries", summ), ("entropies", ent), ("flags", flags)):
            if len(ptrs) != self.nbands:
                raise ValueError(f"{len(ptrs)} peer {name} pointers for {self.nbands} bands")
        self._peer_arrays = tuple(t.tensor([int(p) for p in ptrs], dtype=t.int64, device=self.device)
                                  for ptrs in (hist, summ, ent, flags))

    def attach_peers(self, judges) -> None:
        """Wire this band to the buffers of `judges` (every band, in band
        order) living in this process -- the one-GPU stand-in for the
        symmetric-memory mapping."""
        js = sorted(judges, key=lambda j: j.band)
        if [j.band for j in js] != list(range(self.nbands)):
            raise ValueError("attach_peers needs one judge per band")
        self._set_peer_arrays([j.buf.hist.data_ptr() for j in js], [j.buf.summary.data_ptr() for j in js],
                              [j.buf.ent_all.data_ptr() for j in js], [j.flags.data_ptr() for j in js])

    def next_epoch(self) -> int:
        self._epoch += 1
        return self._epoch

    def _peers(self):
        if self._peer_arrays is None:
            raise RuntimeError("peer exchange without peers: build with exchange='peer' and a group, "
                               "or call attach_peers")
        return self._peer_arrays

    def signal(self, epoch: int, mode: int, stream=None) -> None:
        """pcbz_peer_signal: 1 arrive, 2 wait, 3 both (enqueued)."""
        flags = self._peers()[3]
        _lib.check(_lib.load().pcbz_peer_signal(flags.data_ptr(), self.flags.data_ptr(), self.nbands,
                                                 self.band, ctypes.c_uint32(epoch & 0xFFFFFFFF), mode,
                                                 self._st(stream)))

    def merge_peers(self, stream=None):
        """This rank's slots, pulled from every band over peer memory, scored,
        and their entropies stored into every rank's table."""
        h, sm, en, _ = self._peers()
        rc = _lib.load().pcbz_judge_merge_peers_device(
            self.F, self.H, self.W, self.px, self.py, self.codes.ctypes.data, self.k, self.temporal,
            self.has_halo, self.nbands, self.band, h.data_ptr(), sm.data_ptr(), en.data_ptr(),
            self.buf.hist_owned.data_ptr(), self.buf.ent_owned.data_ptr(), self._st(stream))
        _lib.check(rc)
        return self.buf.ent_owned

    def select(self, stream=None):
        """Every frame's argmin from the gathered entropies."""
        rc = _lib.load().pcbz_judge_select_device(
            self.F, self.codes.ctypes.data, self.k, self.temporal, self.has_halo,
            self.buf.ent_all.data_ptr(), self.sel.data_ptr(), self._st(stream))
        _lib.check(rc)
        return self.sel

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
        """partial -> reduce-scatter / all-to-all -> owned merge -> all-gather
        -> argmin -> emit (shard.band_collective), or with exchange="peer"
        partial -> barrier -> pull-merge-push over peer memory -> barrier ->
        argmin -> emit (shard.band_peer_exchange)."""
        import contextlib

        from .shard import band_collective, band_peer_exchange

        if self.exchange == "peer":
            return band_peer_exchange(self, frames, halo, stream)
        # the collectives order against torch's current stream: run the whole
        # sequence on `stream` as current
        ctx = self.torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            _, sel, out = band_collective(lambda: self.partial(frames, halo, stream),
                                          lambda: self.merge_owned(stream), lambda: self.select(stream),
                                          lambda: self.emit(frames, halo, stream), self.buf, self.nbands,
                                          group)
        return self.ent, sel, out


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
