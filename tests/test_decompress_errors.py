"""decompress_stack error behaviour (reference pipeline.py:121-139,
blocks.py:84-95): an undecodable payload raises BlockDecodeError carrying
the block index (unwrapped); a decodable block of the wrong length raises
CorruptContainerError naming the frame.  Both are raised while decoding,
before any device call, so these run on CPU."""
import bz2
import struct

import numpy as np
import pytest

import oracle
from paper_2310_09467_b200 import BlockDecodeError, CorruptContainerError, decompress_stack
from paper_2310_09467_b200.codec import HEADER_SIZE
from workloads.lfm_synth import SynthParams, generate_array


@pytest.fixture(scope="module")
def container():
    vol = generate_array(SynthParams(24, 20, 4, 4, mode="smooth_lenslet", frames=3, seed=2))
    data, _ = oracle.compress_stack(vol, 4, 4, block_size=300)
    return bytearray(data)


def _layout(data):
    nf = struct.unpack_from("<I", data, 16)[0]
    off, sizes = HEADER_SIZE, []
    for _ in range(nf):
        _, nb = struct.unpack_from("<B3xI", data, off)
        off += 8
        sizes.append(list(struct.unpack_from(f"<{nb}Q", data, off)))
        off += 8 * nb
    return off, sizes


@pytest.mark.parametrize("workers", [1, 4])
def test_bad_payload_raises_block_decode_error(container, workers):
    data = bytearray(container)
    start, sizes = _layout(data)
    off = start + sum(sizes[0]) + sizes[1][0]        # frame 1, block 1
    data[off + 10] ^= 0xFF
    with pytest.raises(BlockDecodeError) as ei:
        decompress_stack(bytes(data), workers=workers)
    assert ei.value.block_index == 1


@pytest.mark.parametrize("workers", [1, 4])
def test_wrong_length_raises_corrupt_container(container, workers):
    data = bytearray(container)
    start, sizes = _layout(data)
    # replace frame 2's last block by a valid bzip2 stream one byte short
    off = start + sum(sizes[0]) + sum(sizes[1]) + sum(sizes[2][:-1])
    raw = bz2.decompress(bytes(data[off:off + sizes[2][-1]]))
    repl = bz2.compress(raw[:-1], 9)
    head_off = HEADER_SIZE + sum(8 + 8 * len(s) for s in sizes[:2]) + 8 + 8 * (len(sizes[2]) - 1)
    struct.pack_into("<Q", data, head_off, len(repl))
    data = data[:off] + repl + data[off + sizes[2][-1]:]
    with pytest.raises(CorruptContainerError, match="frame 2"):
        decompress_stack(bytes(data), workers=workers)
