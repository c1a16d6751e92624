"""Stack compression / decompression around the B200 judge
(reference pkg/src/pcbz/pipeline.py).

compress_stack_detailed keeps the reference's per-frame semantics
(pipeline.py:76-113) but runs them batched: all frames of a chunk are judged
and their selected residual streams emitted by one device call
(pcbz_judge_host), then every (frame, block) pair is bzip2-coded on a host
thread pool while the next chunk is on the GPU.  Output bytes are a pure
function of (stack, options) and identical to the reference's.
"""
from __future__ import annotations

import bz2
import ctypes
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib, criterion
from .codec import (DEFAULT_BLOCK_SIZE, BlockDecodeError, BlockPlan, CompressedBlocks,
                    CorruptContainerError, bz2_block, read_container, split_blocks, write_container)
from .core import Frame, FrameStack, LensletGeometry, PredictorSpec, unpack_symbols
from .criterion import EntropyReport, default_candidates

#: frames per device call in compress_stack (bounded host/device memory)
GPU_CHUNK_FRAMES = 32


@dataclass(frozen=True)
class CompressOptions:
    """Same knobs as reference pipeline.py:26-49."""

    candidates: tuple | None = None
    forced: PredictorSpec | None = None
    block_size: int = DEFAULT_BLOCK_SIZE
    workers: int = 1
    temporal: bool = True
    #: "device": bzip2 on the GPU next to the judge (csrc/bzip2.cu, the same
    #: bytes as libbzip2); "host": bz2.compress on `workers` threads
    coder: str = "device"

    def __post_init__(self):
        if self.coder not in ("device", "host"):
            raise ValueError(f"coder must be 'device' or 'host', got {self.coder!r}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {self.block_size}")
        if self.candidates is not None and not self.candidates:
            raise ValueError("candidate set must not be empty")


@dataclass
class CompressResult:
    data: bytes
    specs: list
    reports: list
    select_seconds: float = 0.0
    encode_seconds: float = 0.0


def candidate_codes(opts: CompressOptions) -> list:
    """Full candidate byte list of a stack (sorted, validated); the device
    drops temporal ones on frames without a previous frame, which is
    reference _frame_candidates (pipeline.py:67-73)."""
    cands = default_candidates(True, opts.temporal) if opts.candidates is None else opts.candidates
    codes = [s.to_byte() for s in cands]
    if len(set(codes)) != len(codes):
        raise ValueError("candidate set contains duplicates")
    if not any(not c & 0x80 for c in codes):
        raise ValueError("no usable candidate for a frame without a previous frame")
    return sorted(codes)


def judge_volume(vol: np.ndarray, geo: LensletGeometry, codes: list, temporal: bool,
                 halo: np.ndarray | None = None, want_stream: bool = True, out=None):
    """One device call: entropies [F, k] (NaN = not scored), selected bytes [F],
    emitted streams [F, 2HW] for a C-contiguous [F, H, W] uint16 volume.
    `out` = (ent, sel, stream) host arrays to fill (e.g. pinned memory)."""
    F, H, W = vol.shape
    spec = np.array(codes, np.uint8)
    if out is not None:
        ent, sel, stream = out
        assert ent.shape == (F, spec.size) and sel.shape == (F,)
        assert stream is None or stream.shape == (F, 2 * H * W)
    else:
        ent = np.empty((F, spec.size), np.float64)
        sel = np.empty(F, np.uint8)
        stream = np.empty((F, 2 * H * W), np.uint8) if want_stream else None
    exact = _lib.ensure_entropy_terms(2 * H * W - 1)
    _lib.check(_lib.load().pcbz_judge_host(
        _lib.ptr(vol), _lib.ptr(halo), F, H, W, geo.pitch_x, geo.pitch_y, _lib.ptr(spec), spec.size,
        1 if temporal else 0, _lib.ptr(ent), _lib.ptr(sel), _lib.ptr(stream)))
    if not exact:
        _guard_near_ties(vol, halo, geo, spec, temporal, ent, sel, stream)
    return ent, sel, stream


def _guard_near_ties(vol, halo, geo, spec, temporal, ent, sel, stream):
    """Near-tie selection guard (criterion.NEAR_TIE_REL) for totals without a
    host term table: re-score those frames with host numpy entropies and
    re-emit a frame whose selection changes."""
    for f in criterion.near_tie_rows(ent):
        prev = (vol[f - 1] if f > 0 else halo) if temporal else None
        scored = ~np.isnan(ent[f])
        e, best = criterion.rescore_on_host(vol[f], prev, spec[scored], geo.pitch_x, geo.pitch_y)
        ent[f, scored] = e
        if best != sel[f]:
            sel[f] = best
            if stream is not None:
                stream[f] = emit_volume(vol[f:f + 1], geo, sel[f:f + 1],
                                        prev if (best & 0x80) else None)[0]


def encode_volume(vol, geo: LensletGeometry, codes, temporal: bool,
                  halo: np.ndarray | None = None, forced_sel: np.ndarray | None = None,
                  block_size: int = DEFAULT_BLOCK_SIZE, views: bool = False):
    """Judge (or the forced modes), emission and bzip2 of every (frame, block)
    on the device (pcbz_compress_host / pcbz_compress_frames_host): (ent [F, k]
    or None, sel [F], payloads [F] of tuples of bzip2 streams).  `vol` is a
    [F, H, W] volume or a sequence of [H, W] frames (passed by pointer, never
    stacked).  Blocks the device leaves to libbzip2 (exactly periodic ones)
    come back raw and are coded here.  views=True returns the payloads as
    memoryviews into one output buffer (no per-block copy; the container
    writer joins them)."""
    frames = None
    if isinstance(vol, np.ndarray) and vol.ndim == 3:
        F, H, W = vol.shape
        vol = np.ascontiguousarray(vol)
    else:
        frames = [np.ascontiguousarray(f, dtype=np.uint16) for f in vol]
        F = len(frames)
        H, W = frames[0].shape
        if any(f.shape != (H, W) for f in frames):
            raise ValueError("all frames must have the same shape")
    lib = _lib.load()
    if forced_sel is None and codes is not None and not _lib.ensure_entropy_terms(2 * H * W - 1):
        # no host term table for this total: judge with the near-tie guard
        # first, then code the selected modes
        v = vol if frames is None else np.stack(frames)
        ent0, sel0, _ = judge_volume(v, geo, list(codes), temporal, halo=halo, want_stream=False)
        _, _, payloads = encode_volume(v, geo, None, temporal, halo, sel0, block_size, views)
        return ent0, sel0, payloads
    nb = -(-2 * H * W // block_size)
    cap = lib.pcbz_compress_bound(F, H, W, block_size)
    # views: payloads land in this thread's page-locked buffer (valid until
    # its next views call); otherwise a fresh array the payloads are copied from
    out = _lib.pinned_buffer(max(cap, 1)) if views else np.empty(max(cap, 1), np.uint8)
    start = np.zeros(F * nb, np.int64)
    length = np.zeros(F * nb, np.int64)
    raw = np.zeros(F * nb, np.uint8)
    spec = None if codes is None else np.array(codes, np.uint8)
    ent = None if forced_sel is not None else np.empty((F, spec.size), np.float64)
    sel = np.empty(F, np.uint8)
    fs = None if forced_sel is None else np.ascontiguousarray(forced_sel, np.uint8)
    tail = (_lib.ptr(halo), F, H, W, geo.pitch_x, geo.pitch_y, _lib.ptr(spec),
            0 if spec is None else spec.size, 1 if temporal else 0, _lib.ptr(fs), block_size,
            _lib.ptr(ent), _lib.ptr(sel), out.ctypes.data, cap, start.ctypes.data, length.ctypes.data,
            raw.ctypes.data)
    if frames is None:
        _lib.check(lib.pcbz_compress_host(_lib.ptr(vol), *tail))
    else:
        ptrs = (ctypes.c_void_p * F)(*[f.ctypes.data for f in frames])
        _lib.check(lib.pcbz_compress_frames_host(ptrs, *tail))
    mv = memoryview(out)
    payloads = []
    for f in range(F):
        blocks = []
        for b in range(nb):
            i = f * nb + b
            piece = mv[start[i]:start[i] + length[i]]
            if raw[i]:
                blocks.append(bz2_block(piece))
            else:
                blocks.append(piece if views else piece.tobytes())
        payloads.append(tuple(blocks))
    return ent, sel, payloads


def emit_volume(vol: np.ndarray, geo: LensletGeometry, sel: np.ndarray,
                halo: np.ndarray | None = None) -> np.ndarray:
    F, H, W = vol.shape
    s = np.ascontiguousarray(sel, dtype=np.uint8)
    stream = np.empty((F, 2 * H * W), np.uint8)
    _lib.check(_lib.load().pcbz_emit_host(_lib.ptr(vol), _lib.ptr(halo), F, H, W, geo.pitch_x,
                                          geo.pitch_y, _lib.ptr(s), _lib.ptr(stream)))
    return stream


def _reports(ent: np.ndarray, codes: list) -> list:
    out = []
    for row in ent:
        entries = tuple((PredictorSpec.from_byte(c), float(e)) for c, e in zip(codes, row)
                        if not np.isnan(e))
        best = min(entries, key=lambda se: (se[1], se[0].to_byte()))
        out.append(EntropyReport(entries=entries, selected=best[0]))
    return out


def compress_stack_detailed(stack: FrameStack, opts: CompressOptions | None = None) -> CompressResult:
    """Reference pipeline.py:76-113 semantics, batched on the device."""
    opts = opts or CompressOptions()
    geo = stack.geometry
    F = stack.frame_count
    forced = opts.forced
    codes = None if forced is not None else candidate_codes(opts)
    specs, reports = [], []
    payloads = [None] * F
    select_s = encode_s = 0.0
    if opts.coder == "device":
        # one call over frame pointers (the library rounds the volume through
        # the device in <= 1 GiB pieces); payloads stay views into its output
        # buffer until the container join copies them once
        t0 = time.perf_counter()
        fsel = None
        if forced is not None:
            fsel = np.array([forced.to_byte() if (i > 0 and opts.temporal) else forced.intra_id
                             for i in range(F)], np.uint8)
        ent, sel, pl = encode_volume([f.samples for f in stack.frames], geo, codes, opts.temporal, None,
                                     fsel, opts.block_size, views=True)
        encode_s = time.perf_counter() - t0
        reports = _reports(ent, codes) if forced is None else [None] * F
        specs = [PredictorSpec.from_byte(int(c)) for c in sel]
        payloads = [CompressedBlocks(BlockPlan(opts.block_size, len(p)), p) for p in pl]
        data = write_container(stack.width, stack.height, geo.pitch_x, geo.pitch_y, opts.block_size,
                               list(zip(specs, payloads)), joiner=_lib.join)
        return CompressResult(data, specs, reports, select_s, encode_s)
    vol = np.ascontiguousarray(stack.to_array())
    pool = ThreadPoolExecutor(max(1, opts.workers))
    futures = []
    try:
        for a in range(0, F, GPU_CHUNK_FRAMES):
            b = min(F, a + GPU_CHUNK_FRAMES)
            chunk = vol[a:b]
            halo = vol[a - 1] if (a > 0 and opts.temporal) else None
            t0 = time.perf_counter()
            if forced is None:
                ent, sel, streams = judge_volume(chunk, geo, codes, opts.temporal, halo)
                reports += _reports(ent, codes)
                select_s += time.perf_counter() - t0
            else:
                sel = np.array([forced.to_byte() if (a + i > 0 and opts.temporal) else forced.intra_id
                                for i in range(b - a)], np.uint8)
                streams = emit_volume(chunk, geo, sel, halo)
                reports += [None] * (b - a)
                encode_s += time.perf_counter() - t0
            specs += [PredictorSpec.from_byte(int(c)) for c in sel]
            for i in range(b - a):
                for j, blk in enumerate(split_blocks(streams[i], opts.block_size)):
                    futures.append((a + i, j, pool.submit(bz2_block, blk)))
        t0 = time.perf_counter()
        by_frame = {}
        for fi, j, fut in futures:
            by_frame.setdefault(fi, []).append(fut.result())
        encode_s += time.perf_counter() - t0
    finally:
        pool.shutdown(wait=True)
    for fi in range(F):
        blocks = by_frame.get(fi, [])
        payloads[fi] = CompressedBlocks(BlockPlan(opts.block_size, len(blocks)), tuple(blocks))
    data = write_container(stack.width, stack.height, geo.pitch_x, geo.pitch_y, opts.block_size,
                           list(zip(specs, payloads)))
    return CompressResult(data, specs, reports, select_s, encode_s)


def compress_stack(stack: FrameStack, opts: CompressOptions | None = None) -> bytes:
    return compress_stack_detailed(stack, opts).data


class _done:
    """An already-available result with the Future.result() interface."""

    def __init__(self, value):
        self.value = value

    def result(self):
        return self.value


@dataclass
class StreamResult:
    frames: int
    container_bytes: int
    specs: list
    select_seconds: float = 0.0
    encode_wait_seconds: float = 0.0


def compress_stream(frames, geometry: LensletGeometry, out, opts: CompressOptions | None = None,
                    nframes: int | None = None, chunk_frames: int = GPU_CHUNK_FRAMES,
                    max_inflight_chunks: int = 3, judge_fn=None) -> StreamResult:
    """Bounded-memory compress_stack for long series:
    `frames` is any iterable of 2-D uint16 arrays (or Frames) of one shape;
    the container goes to the binary file `out` and is byte-identical to
    compress_stack on the same frames (reference pipeline.py:76-113).
    Chunks of `chunk_frames` frames are judged and emitted by one device call
    (the previous chunk's last frame is the temporal halo); their bzip2
    blocks are coded on `opts.workers` threads while the next chunks are
    read and judged, with at most `max_inflight_chunks` chunks of streams
    alive.  `judge_fn(chunk, halo, geo, codes, temporal) -> (ent, sel,
    streams)` defaults to the device judge (tests inject the oracle)."""
    from .codec import ContainerWriter
    opts = opts or CompressOptions()
    forced = opts.forced
    codes = None if forced is not None else candidate_codes(opts)
    injected = judge_fn
    if judge_fn is None:
        def judge_fn(chunk, halo, geo, cands, temporal):
            return judge_volume(chunk, geo, cands, temporal, halo=halo)
    pool = ThreadPoolExecutor(max(1, opts.workers))
    writer = None
    specs = []
    pending = []          # [(spec, [futures])] in frame order
    halo = None
    select_s = wait_s = 0.0
    nseen = 0

    def drain(keep_chunks: int):
        nonlocal wait_s
        while len(pending) > keep_chunks:
            t0 = time.perf_counter()
            for spec, futs in pending.pop(0):
                writer.add_frame(spec, [f.result() for f in futs])
            wait_s += time.perf_counter() - t0

    device_coder = opts.coder == "device" and injected is None

    def run_chunk(buf):
        nonlocal halo, select_s
        chunk = np.ascontiguousarray(np.stack(buf))
        h = halo if opts.temporal else None
        t0 = time.perf_counter()
        if device_coder:
            first = nseen - len(buf)
            fsel = None if forced is None else np.array(
                [forced.to_byte() if (first + i > 0 and opts.temporal) else forced.intra_id
                 for i in range(len(buf))], np.uint8)
            _, sel, pl = encode_volume(chunk, geometry, codes, opts.temporal, h, fsel, opts.block_size)
            select_s += time.perf_counter() - t0
            halo = chunk[-1].copy()
            entry = []
            for i in range(len(buf)):
                spec = PredictorSpec.from_byte(int(sel[i]))
                specs.append(spec)
                entry.append((spec, [_done(p) for p in pl[i]]))
            pending.append(entry)
            drain(max_inflight_chunks - 1)
            return
        if forced is None:
            _, sel, streams = judge_fn(chunk, h, geometry, codes, opts.temporal)
        else:
            first = nseen - len(buf)
            sel = np.array([forced.to_byte() if (first + i > 0 and opts.temporal) else forced.intra_id
                            for i in range(len(buf))], np.uint8)
            streams = emit_volume(chunk, geometry, sel, h)
        select_s += time.perf_counter() - t0
        halo = chunk[-1].copy()
        entry = []
        for i in range(len(buf)):
            spec = PredictorSpec.from_byte(int(sel[i]))
            specs.append(spec)
            entry.append((spec, [pool.submit(bz2_block, blk)
                                 for blk in split_blocks(streams[i], opts.block_size)]))
        pending.append(entry)
        drain(max_inflight_chunks - 1)

    try:
        buf = []
        for fr in frames:
            a = fr.samples if isinstance(fr, Frame) else np.asarray(fr)
            if a.dtype != np.uint16 or a.ndim != 2:
                raise ValueError("frames must be 2-D uint16 arrays")
            if writer is None:
                H, W = a.shape
                writer = ContainerWriter(out, W, H, geometry.pitch_x, geometry.pitch_y,
                                         opts.block_size, nframes)
            elif a.shape != (H, W):
                raise ValueError(f"frame {nseen} has shape {a.shape}, expected {(H, W)}")
            buf.append(a)
            nseen += 1
            if len(buf) == chunk_frames:
                run_chunk(buf)
                buf = []
        if buf:
            run_chunk(buf)
        if writer is None:
            raise ValueError("container must hold at least one frame")
        drain(0)
        size = writer.close()
    finally:
        pool.shutdown(wait=True)
    return StreamResult(nseen, size, specs, select_s, wait_s)


def decompress_stack(data, workers: int = 1) -> FrameStack:
    """Reference pipeline.py:121-139: bzip2 on host threads, inverse
    prediction and temporal undelta on the device."""
    header, records, payloads = read_container(data)
    fast = None
    if _lib.device_count() > 0 and _prefer_device_decode(header, payloads, workers):
        fast = _decompress_device(header, records, payloads)
    if fast is not None:
        return fast
    # anything the device decoder leaves to libbzip2 (corrupt or unusual
    # payloads): the whole container takes the host path below, which raises
    # the reference's errors in frame order
    H, W = header.height, header.width
    res = np.empty((header.frame_count, H, W), np.uint16)
    # every (frame, block) payload of the container on one pool (the
    # reference decodes frame by frame, pipeline.py:127-133, which leaves all
    # but block_count threads idle); errors are reported for the first bad
    # frame in frame order, as the sequential loop would
    jobs = [(j, bytes(p)) for i in range(len(records)) for j, p in enumerate(payloads[i])]

    def decode(job):
        j, payload = job
        try:
            return bz2.decompress(payload), None
        except (OSError, EOFError, ValueError) as exc:   # codec.decompress_blocks' mapping
            return None, BlockDecodeError(j, str(exc))

    if workers > 1 and len(jobs) > 1:
        with ThreadPoolExecutor(workers) as pool:
            decoded = list(pool.map(decode, jobs))
    else:
        decoded = [decode(j) for j in jobs]
    k = 0
    for i, rec in enumerate(records):
        parts = decoded[k:k + len(payloads[i])]
        k += len(payloads[i])
        for _, exc in parts:    # undecodable payload: BlockDecodeError, unwrapped (blocks.py:87-92)
            if exc is not None:
                raise exc
        try:
            res[i] = unpack_symbols(b"".join(p for p, _ in parts), W, H)
        except ValueError as exc:
            raise CorruptContainerError(f"frame {i}: {exc}") from exc
    sel = np.array([r.spec.to_byte() for r in records], np.uint8)
    out = np.empty_like(res)
    # inverse prediction in rounds of <= DECOMPRESS_ROUND_BYTES of frames (a
    # round's first frame reads the previous round's last reconstructed one)
    per = max(1, DECOMPRESS_ROUND_BYTES // (2 * H * W))
    for a in range(0, res.shape[0], per):
        b = min(res.shape[0], a + per)
        _lib.check(_lib.load().pcbz_reconstruct_host(
            _lib.ptr(res[a:b]), _lib.ptr(out[a - 1]) if a > 0 else None, b - a, H, W,
            header.pitch_x, header.pitch_y, _lib.ptr(np.ascontiguousarray(sel[a:b])), _lib.ptr(out[a:b])))
    geo = LensletGeometry(header.pitch_x, header.pitch_y)
    return FrameStack(tuple(Frame(f, geo) for f in out))


def _prefer_device_decode(header, payloads, workers: int) -> bool:
    """The device decoder's time is set by its slowest block (one warp runs a
    block's Huffman + MTF: ~0.25 s per 900 KB block, measured), the host
    pool's by payloads per thread (libbzip2 ~23 MB/s per thread): small
    containers decode faster on host threads."""
    n = sum(len(p) for p in payloads)
    raw = 2 * header.width * header.height * header.frame_count
    gpu_s = 0.25 + raw / 2.0e9
    host_s = -(-n // max(1, workers)) * min(header.block_size, 2 * header.width * header.height) / 23e6
    return gpu_s < host_s


#: decoded bytes per pcbz_decompress_host round (bounds device and page-locked memory)
DECOMPRESS_ROUND_BYTES = 1 << 30


def _decompress_device(header, records, payloads):
    """Every payload bzip2-decoded on the GPU (pcbz_decompress_host: block
    magic scan, Huffman + inverse MTF, inverse BWT by list ranking, inverse
    RLE1, all CRCs checked) and the inverse prediction run on the decoded
    streams without leaving the device, in rounds of <= 1 GiB of frames (a
    round's temporal first frame reads the previous round's last frame).
    None when any payload or the block layout is not the one compress_stack
    writes (the caller's host path then decodes and reports errors exactly as
    the reference)."""
    H, W = header.height, header.width
    F = header.frame_count
    nb = -(-2 * H * W // header.block_size)
    if any(len(p) != nb for p in payloads):
        return None
    sel_all = np.array([r.spec.to_byte() for r in records], np.uint8)
    out = np.empty((F, H, W), np.uint16)
    per = max(1, DECOMPRESS_ROUND_BYTES // (2 * H * W))
    lib = _lib.load()
    for a in range(0, F, per):
        b = min(F, a + per)
        flat = [p for ps in payloads[a:b] for p in ps]
        n = len(flat)
        ptrs = (ctypes.c_void_p * n)(*[_lib._address(p) for p in flat])
        lens = np.array([len(p) for p in flat], np.int64)
        sel = np.ascontiguousarray(sel_all[a:b])
        status = np.ones(n, np.uint8)
        # frames land in this thread's page-locked buffer (PCIe speed), then a
        # multithreaded copy moves them into the returned array
        staged = _lib.pinned_buffer((b - a) * H * W * 2)
        halo = out[a - 1] if a > 0 else None
        rc = lib.pcbz_decompress_host(ptrs, lens.ctypes.data, b - a, nb, H, W, header.pitch_x,
                                      header.pitch_y, header.block_size, _lib.ptr(sel), _lib.ptr(halo),
                                      None, staged.ctypes.data, status.ctypes.data)
        if rc == _lib.PCBZ_NEEDS_HOST:
            # blocks the device leaves to libbzip2 (e.g. exactly periodic
            # ones): decode only those here and call again with them
            host = _host_decode_blocks(flat, status, nb, 2 * H * W, header.block_size)
            if host is None:    # a real decode error: the host path reports it
                return None
            hs = (ctypes.c_void_p * n)(*[None if d is None else _lib._address(d) for d in host])
            rc = lib.pcbz_decompress_host(ptrs, lens.ctypes.data, b - a, nb, H, W, header.pitch_x,
                                          header.pitch_y, header.block_size, _lib.ptr(sel), _lib.ptr(halo),
                                          hs, staged.ctypes.data, status.ctypes.data)
            if rc == _lib.PCBZ_NEEDS_HOST:
                return None
        _lib.check(rc)
        _lib.copy_into(out[a:b], staged)
    geo = LensletGeometry(header.pitch_x, header.pitch_y)
    return FrameStack(tuple(Frame(f, geo) for f in out))


def _host_decode_blocks(flat, status, nb: int, stream_bytes: int, block_size: int):
    """libbzip2 on host threads for the payloads with status 1: a list with
    the decoded bytes at those positions (None elsewhere), or None when one
    of them does not decode to its block's length."""
    need = [int(i) for i in np.nonzero(status)[0]]

    def one(i):
        try:
            d = bz2.decompress(bytes(flat[i]))
        except (OSError, EOFError, ValueError):
            return None
        want = min(block_size, stream_bytes - (i % nb) * block_size)
        return d if len(d) == want else None

    with ThreadPoolExecutor(min(len(need), 16) or 1) as pool:
        got = list(pool.map(one, need))
    if any(d is None for d in got):
        return None
    host = [None] * len(flat)
    for i, d in zip(need, got):
        host[i] = d
    return host


@dataclass
class Metrics:
    uncompressed_bytes: int
    container_bytes: int
    compression_ratio: float
    bits_per_dim: float
    compress_seconds: float | None = None
    decompress_seconds: float | None = None


def measure(container: bytes, stack: FrameStack, compress_seconds=None, decompress_seconds=None):
    """Reference pipeline.py:154-168."""
    n = stack.width * stack.height * stack.frame_count
    return Metrics(stack.nbytes, len(container), stack.nbytes / len(container),
                   8.0 * len(container) / n, compress_seconds, decompress_seconds)
