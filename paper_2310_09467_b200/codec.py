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
                    frames: Sequence) -> bytes:
    """Header, per-frame records, then payloads in frame/block order
    (container.py:84-106, FORMAT.md)."""
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
    return b"".join(parts)


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
