"""Host back end kept unchanged from the reference: fixed-size bzip2 blocks and
the PCBZ container (reference pkg/src/pcbz/blocks.py, container.py,
pkg/FORMAT.md).  Written here so the package is standalone on machines
without `pcbz`; output bytes are identical by construction (same libbz2 call,
same little-endian layout) and pinned by container hashes from the reference
in tests/golden.
"""
from __future__ import annotations

import bz2
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Sequence

from .core import PredictorSpec

DEFAULT_BLOCK_SIZE = 4 * 1024 * 1024      # blocks.py:20
BZ2_LEVEL = 9                             # blocks.py:21
MAGIC = b"PCBZ"
VERSION = 1
BIT_DEPTH = 16
FLAG_TEMPORAL = 0x01
_HEAD = struct.Struct("<4sBBBBIIIHHI")    # 28 bytes, container.py:41
_REC = struct.Struct("<B3xI")             # 8 bytes, container.py:42
HEADER_SIZE = _HEAD.size


class PcbzError(Exception):
    """Base of the data errors (reference errors.py:10-41)."""


class ContainerFormatError(PcbzError):
    pass


class NotAContainerError(ContainerFormatError):
    pass


class CorruptContainerError(ContainerFormatError):
    pass


class BlockDecodeError(PcbzError):
    def __init__(self, block_index: int, message: str = ""):
        self.block_index = block_index
        super().__init__(f"block {block_index}: {message or 'payload is not a valid bzip2 stream'}")


@dataclass(frozen=True)
class BlockPlan:
    block_size: int
    block_count: int

    @classmethod
    def for_length(cls, length: int, block_size: int) -> "BlockPlan":
        if block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {block_size}")
        return cls(block_size, -(-length // block_size) if length else 0)


@dataclass(frozen=True)
class CompressedBlocks:
    plan: BlockPlan
    payloads: tuple

    @property
    def compressed_sizes(self) -> tuple:
        return tuple(len(p) for p in self.payloads)


def split_blocks(stream, block_size: int) -> list:
    mv = memoryview(stream)
    n = BlockPlan.for_length(len(mv), block_size).block_count
    return [mv[i * block_size:(i + 1) * block_size] for i in range(n)]


def bz2_block(chunk) -> bytes:
    return bz2.compress(chunk, BZ2_LEVEL)


def bunzip2_blocks_device(payloads, sizes) -> list:
    """bz2.decompress of every payload (whose decoded size is known: PCBZ
    blocks), decoded on the GPU by csrc/bunzip2.cu (pcbz_bunzip2_host); a
    payload the device leaves to libbzip2 (status 1) is decoded on the host."""
    import ctypes
    import numpy as np
    from . import _lib
    n = len(payloads)
    if n == 0:
        return []
    ptrs = (ctypes.c_void_p * n)(*[_lib._address(p) if len(p) else None for p in payloads])
    lens = np.array([len(p) for p in payloads], np.int64)
    osz = np.array(sizes, np.int64)
    off = np.zeros(n, np.int64)
    off[1:] = np.cumsum(osz)[:-1]
    out = np.empty(max(int(osz.sum()), 1), np.uint8)
    status = np.ones(n, np.uint8)
    _lib.check(_lib.load().pcbz_bunzip2_host(ptrs, lens.ctypes.data, n, out.ctypes.data, off.ctypes.data,
                                             osz.ctypes.data, status.ctypes.data))
    return [out[off[i]:off[i] + osz[i]].tobytes() if status[i] == 0 else bz2.decompress(payloads[i])
            for i in range(n)]


#: input bytes per pcbz_bzip2_host call (the device coder takes < 2^31 bytes after RLE1)
DEVICE_BZ2_BATCH = 1 << 30


def bz2_blocks_device(chunks) -> list:
    """bz2.compress(chunk, 9) of every chunk, coded on the GPU by
    csrc/bzip2.cu (pcbz_bzip2_host), byte-exact with libbzip2 1.0.8.  A chunk
    holding an exactly periodic block -- whose rotation ties libbzip2 breaks
    in an implementation-defined order -- is coded by the host libbzip2."""
    import numpy as np

    from . import _lib
    lib = _lib.load()
    chunks = [memoryview(c).cast("B") for c in chunks]
    out_all, i = [], 0
    while i < len(chunks):
        j, size = i, 0
        while j < len(chunks) and (j == i or size + len(chunks[j]) <= DEVICE_BZ2_BATCH):
            size += len(chunks[j])
            j += 1
        batch = chunks[i:j]
        off = np.zeros(len(batch) + 1, np.int64)
        off[1:] = np.cumsum([len(c) for c in batch])
        buf = np.empty(max(int(off[-1]), 1), np.uint8)
        for k, c in enumerate(batch):
            buf[off[k]:off[k + 1]] = np.frombuffer(c, np.uint8)
        cap = lib.pcbz_bzip2_bound(off.ctypes.data, len(batch))
        out = np.empty(max(cap, 1), np.uint8)
        start = np.zeros(len(batch), np.int64)
        length = np.zeros(len(batch), np.int64)
        host = np.zeros(len(batch), np.uint8)
        rc = lib.pcbz_bzip2_host(buf.ctypes.data, off.ctypes.data, len(batch), out.ctypes.data, cap,
                                 start.ctypes.data, length.ctypes.data, host.ctypes.data)
        if rc:
            msg = lib.pcbz_bzip2_last_error().decode(errors="replace")
            raise (ValueError if rc == _lib.PCBZ_E_INVALID else RuntimeError)(msg)
        for k, c in enumerate(batch):
            out_all.append(bz2.compress(c, BZ2_LEVEL) if host[k]
                           else out[start[k]:start[k] + length[k]].tobytes())
        i = j
    return out_all


def compress_blocks(stream, block_size: int = DEFAULT_BLOCK_SIZE, workers: int = 1) -> CompressedBlocks:
    """blocks.py:73-81: every block is an independent level-9 bzip2 stream."""
    chunks = split_blocks(stream, block_size)
    if workers > 1 and len(chunks) > 1:
        with ThreadPoolExecutor(workers) as pool:
            payloads = list(pool.map(bz2_block, chunks))
    else:
        payloads = [bz2_block(c) for c in chunks]
    return CompressedBlocks(BlockPlan(block_size, len(chunks)), tuple(payloads))


def decompress_blocks(blocks: CompressedBlocks, workers: int = 1) -> bytes:
    def one(item):
        i, payload = item
        try:
            return bz2.decompress(payload)
        except (OSError, EOFError, ValueError) as exc:
            raise BlockDecodeError(i, str(exc)) from exc
    items = list(enumerate(blocks.payloads))
    if workers > 1 and len(items) > 1:
        with ThreadPoolExecutor(workers) as pool:
            return b"".join(pool.map(one, items))
    return b"".join(one(i) for i in items)


@dataclass(frozen=True)
class ContainerHeader:
    width: int
    height: int
    frame_count: int
    pitch_x: int
    pitch_y: int
    block_size: int
    temporal_used: bool = False


@dataclass(frozen=True)
class FrameRecord:
    spec: PredictorSpec
    block_sizes: tuple


def write_container(width: int, height: int, pitch_x: int, pitch_y: int, block_size: int,
                    frames: Sequence, joiner=None) -> bytes:
    """Header, per-frame records, then payloads in frame/block order
    (container.py:84-106, FORMAT.md).  `joiner` replaces b"".join (the
    device path passes the native multithreaded join, _lib.join)."""
    frames = list(frames)
    if not frames:
        raise ValueError("container must hold at least one frame")
    if frames[0][0].temporal:
        raise ValueError("frame 0 must not use a temporal predictor")
    flags = FLAG_TEMPORAL if any(s.temporal for s, _ in frames) else 0
    parts = [_HEAD.pack(MAGIC, VERSION, flags, BIT_DEPTH, 0, width, height, len(frames),
                        pitch_x, pitch_y, block_size)]
    for spec, blocks in frames:
        sizes = blocks.compressed_sizes
        parts.append(_REC.pack(spec.to_byte(), len(sizes)))
        parts.append(struct.pack(f"<{len(sizes)}Q", *sizes))
    for _, blocks in frames:
        parts.extend(blocks.payloads)
    return joiner(parts) if joiner else b"".join(parts)


class ContainerWriter:
    """Incremental writer of the same bytes write_container produces, for
    series too long to hold in memory.  Payloads are
    appended as frames complete; the header (frame count, temporal flag) and
    the per-frame records (compressed block sizes) are written at close().
    With a known frame count and a seekable output, header and record space
    is reserved up front and patched in place; otherwise payloads are spooled
    to a temporary file and copied behind the header at close()."""

    def __init__(self, out, width: int, height: int, pitch_x: int, pitch_y: int, block_size: int,
                 nframes: int | None = None):
        import tempfile
        if min(width, height, pitch_x, pitch_y, block_size) < 1:
            raise ValueError("non-positive container field")
        self.out = out
        self.dims = (width, height, pitch_x, pitch_y, block_size)
        self.blocks_per_frame = BlockPlan.for_length(2 * width * height, block_size).block_count
        self.nframes = nframes
        self.records = []
        self.temporal = False
        seekable = getattr(out, "seekable", lambda: False)()
        if nframes is not None and nframes >= 1 and seekable:
            self.base = out.tell()
            self.reserved = HEADER_SIZE + nframes * (_REC.size + 8 * self.blocks_per_frame)
            out.write(b"\0" * self.reserved)
            self.spool = None
        else:
            self.spool = tempfile.TemporaryFile()
        self.closed = False

    def add_frame(self, spec, payloads) -> None:
        if self.closed:
            raise ValueError("container writer is closed")
        if not self.records and spec.temporal:
            raise ValueError("frame 0 must not use a temporal predictor")
        if self.nframes is not None and len(self.records) >= self.nframes:
            raise ValueError(f"more than the announced {self.nframes} frames")
        if len(payloads) != self.blocks_per_frame:
            raise ValueError(f"frame has {len(payloads)} blocks, expected {self.blocks_per_frame}")
        dst = self.spool if self.spool is not None else self.out
        for p in payloads:
            dst.write(p)
        self.records.append((spec.to_byte(), tuple(len(p) for p in payloads)))
        self.temporal |= bool(spec.temporal)

    def _head_and_records(self) -> bytes:
        w, h, px, py, bs = self.dims
        parts = [_HEAD.pack(MAGIC, VERSION, FLAG_TEMPORAL if self.temporal else 0, BIT_DEPTH, 0,
                            w, h, len(self.records), px, py, bs)]
        for code, sizes in self.records:
            parts.append(_REC.pack(code, len(sizes)))
            parts.append(struct.pack(f"<{len(sizes)}Q", *sizes))
        return b"".join(parts)

    def close(self) -> int:
        """Finish the container; returns its size in bytes."""
        import shutil
        if self.closed:
            raise ValueError("container writer is closed")
        if not self.records:
            raise ValueError("container must hold at least one frame")
        if self.nframes is not None and len(self.records) != self.nframes:
            raise ValueError(f"{len(self.records)} frames written, {self.nframes} announced")
        head = self._head_and_records()
        payload_bytes = sum(sum(sz) for _, sz in self.records)
        if self.spool is None:
            assert len(head) == self.reserved
            end = self.out.tell()
            self.out.seek(self.base)
            self.out.write(head)
            self.out.seek(end)
        else:
            self.out.write(head)
            self.spool.seek(0)
            shutil.copyfileobj(self.spool, self.out, 16 << 20)
            self.spool.close()
        self.closed = True
        return len(head) + payload_bytes


def read_container(data):
    """Parse and validate (container.py:109-177); returns (header, records, payloads)."""
    buf = memoryview(data)
    if len(buf) < 4 or bytes(buf[:4]) != MAGIC:
        raise NotAContainerError(f"bad magic {bytes(buf[:4])!r}, expected {MAGIC!r}")
    if len(buf) < HEADER_SIZE:
        raise CorruptContainerError(f"truncated header: {len(buf)} bytes, need {HEADER_SIZE}")
    _, ver, flags, depth, _, w, h, nf, px, py, bs = _HEAD.unpack_from(buf, 0)
    if ver != VERSION:
        raise ContainerFormatError(f"unsupported container version {ver}")
    if depth != BIT_DEPTH:
        raise ContainerFormatError(f"unsupported bit depth {depth}")
    if min(w, h, nf, px, py, bs) < 1:
        raise CorruptContainerError("non-positive header field")
    header = ContainerHeader(w, h, nf, px, py, bs, bool(flags & FLAG_TEMPORAL))
    off, records = HEADER_SIZE, []
    for fi in range(nf):
        if off + _REC.size > len(buf):
            raise CorruptContainerError(f"truncated record for frame {fi} at offset {off}")
        code, nb = _REC.unpack_from(buf, off)
        off += _REC.size
        try:
            spec = PredictorSpec.from_byte(code)
        except ValueError as exc:
            raise CorruptContainerError(f"frame {fi}: {exc}") from exc
        if fi == 0 and spec.temporal:
            raise CorruptContainerError("frame 0 carries a temporal predictor flag")
        if off + 8 * nb > len(buf):
            raise CorruptContainerError(f"truncated block table for frame {fi} at offset {off}")
        records.append(FrameRecord(spec, struct.unpack_from(f"<{nb}Q", buf, off)))
        off += 8 * nb
    payloads = []
    for fi, rec in enumerate(records):
        cur = []
        for bi, size in enumerate(rec.block_sizes):
            if off + size > len(buf):
                raise CorruptContainerError(f"payload truncated in frame {fi} block {bi}")
            cur.append(buf[off:off + size])
            off += size
        payloads.append(cur)
    if off != len(buf):
        raise CorruptContainerError(f"{len(buf) - off} trailing bytes after payload region")
    return header, records, payloads
