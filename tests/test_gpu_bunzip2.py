"""GPU bzip2 decoding (csrc/bunzip2.cu via codec.bunzip2_blocks_device and
pcbz_bunzip2_host) against the reference's bz2.decompress (blocks.py:84-92):
identical bytes for small, multi-block, every-level and run-heavy streams;
payloads the decoder leaves to libbzip2 (periodic blocks, corruption) still
come out right or raise as the reference does; decompress_stack round trip
through the all-device path."""
import bz2
import ctypes
import random

import numpy as np
import pytest

from paper_2310_09467_b200 import _lib
from paper_2310_09467_b200.codec import bunzip2_blocks_device
from workloads.lfm_synth import SynthParams, generate_array

pytestmark = pytest.mark.gpu


def _status(payloads, sizes):
    n = len(payloads)
    ptrs = (ctypes.c_void_p * n)(*[_lib._address(p) for p in payloads])
    lens = np.array([len(p) for p in payloads], np.int64)
    osz = np.array(sizes, np.int64)
    off = np.zeros(n, np.int64)
    off[1:] = np.cumsum(osz)[:-1]
    out = np.empty(max(int(osz.sum()), 1), np.uint8)
    st = np.ones(n, np.uint8)
    _lib.check(_lib.load().pcbz_bunzip2_host(ptrs, lens.ctypes.data, n, out.ctypes.data, off.ctypes.data,
                                             osz.ctypes.data, st.ctypes.data))
    return st, [out[off[i]:off[i] + osz[i]].tobytes() for i in range(n)]


def _periodic(c):
    return any(len(c) % p == 0 and c == c[:p] * (len(c) // p) for p in range(1, len(c)))


def _cases(seed, count):
    rng = random.Random(seed)
    out = [b"", b"a", b"ab", b"banana", b"abcd" * 3, bytes(range(256)), b"aaaab", b"aaaaab",
           b"xaaaa" * 7 + b"y", bytes(rng.randrange(256) for _ in range(5000))]
    for _ in range(count):
        n = rng.choice([3, 9, 17, 100, 700, 2000, 20000, 120000])
        alph = rng.choice([2, 3, 16, 256])
        s = bytearray()
        while len(s) < n:
            s += bytes([rng.randrange(alph)]) * (rng.randint(1, 300) if rng.random() < 0.1 else rng.randint(1, 6))
        out.append(bytes(s[:n]))
    return out


def test_small_streams_identical():
    cases = _cases(5, 120)
    payloads = [bz2.compress(c, 9) for c in cases]
    st, got = _status(payloads, [len(c) for c in cases])
    for c, g, s in zip(cases, got, st):
        if s == 0:
            assert g == c, (len(c), c[:24])
        else:   # only exactly periodic blocks ("xxx", "abcd" * 3) are left to the host
            assert _periodic(c), (len(c), c[:24])
    assert (st == 0).mean() > 0.8
    assert bunzip2_blocks_device(payloads, [len(c) for c in cases]) == cases


@pytest.mark.parametrize("level", [1, 5, 9])
def test_levels_and_multiblock(level):
    rng = np.random.default_rng(level)
    data = (rng.normal(0, 30, 3_000_000).astype(np.int16).astype(np.uint16)).tobytes()
    runs = bytes(np.repeat(rng.integers(0, 256, 40000, dtype=np.uint8), rng.integers(1, 40, 40000)))
    cases = [data, runs[:2_500_000], data[:1_000_001]]
    payloads = [bz2.compress(c, level) for c in cases]
    st, got = _status(payloads, [len(c) for c in cases])
    assert list(st) == [0, 0, 0]
    assert got == cases


def test_residual_streams_like_the_pipeline():
    img = generate_array(SynthParams(2048, 2048, 15, 15, mode="beads", signal_amplitude=3000,
                                     noise_sigma=100, photon_scale=0.05, seed=2))[0]
    from paper_2310_09467_b200.codec import split_blocks
    stream = img.astype(">u2").tobytes()
    chunks = [bytes(b) for b in split_blocks(stream, 4 << 20)]
    payloads = [bz2.compress(c, 9) for c in chunks]
    st, got = _status(payloads, [len(c) for c in chunks])
    assert list(st) == [0] * len(chunks)
    assert got == chunks


def test_periodic_and_corrupt_payloads_left_to_libbzip2():
    const = b"\x07" * (255 * 4000)             # RLE1: (07 07 07 07 FB) x 4000, an exactly periodic block
    good = bytes(np.random.default_rng(1).integers(0, 7, 200_000, dtype=np.uint8))
    p_const, p_good = bz2.compress(const, 9), bz2.compress(good, 9)
    bad = bytearray(p_good)
    bad[len(bad) // 2] ^= 0x40
    st, got = _status([p_const, p_good, bytes(bad)], [len(const), len(good), len(good)])
    assert st[0] == 1 and st[1] == 0 and st[2] == 1
    assert got[1] == good
    assert bunzip2_blocks_device([p_const, p_good], [len(const), len(good)]) == [const, good]
    with pytest.raises((OSError, ValueError, EOFError)):
        bunzip2_blocks_device([bytes(bad)], [len(good)])


def test_device_decode_chosen_for_large_containers():
    """Small containers decode faster on host threads (one slow warp per
    block vs libbzip2 per thread); the device decoder takes large ones."""
    from paper_2310_09467_b200 import pipeline
    from paper_2310_09467_b200.codec import ContainerHeader
    big = ContainerHeader(2048, 2048, 100, 15, 15, 4 << 20, False)
    small = ContainerHeader(2048, 2048, 1, 15, 15, 4 << 20, False)
    assert pipeline._prefer_device_decode(big, [[b"x", b"y"]] * 100, 16)
    assert not pipeline._prefer_device_decode(small, [[b"x", b"y"]], 16)


def test_decompress_stack_device_path_round_trip():
    from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry,
                                       compress_stack, decompress_stack, pipeline)
    p = SynthParams(512, 384, 15, 15, mode="smooth_lenslet", noise_sigma=20.0, photon_scale=0.05,
                    frames=4, drift=1.0, seed=4)
    vol = generate_array(p)
    stack = FrameStack(tuple(Frame(f, LensletGeometry(15, 15)) for f in vol))
    data = compress_stack(stack, CompressOptions(block_size=100_000))
    from paper_2310_09467_b200.codec import read_container
    h, r, pl = read_container(data)
    fast = pipeline._decompress_device(h, r, pl)
    assert fast is not None and fast == stack
    assert decompress_stack(data) == stack


def test_decompress_rounds_carry_the_temporal_halo(monkeypatch):
    """Rounds of frames (DECOMPRESS_ROUND_BYTES): a round's temporal first
    frame is reconstructed from the previous round's last frame."""
    from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry,
                                       compress_stack, decompress_stack, pipeline)
    p = SynthParams(256, 160, 15, 15, mode="smooth_lenslet", noise_sigma=10.0, photon_scale=0.05,
                    frames=7, drift=1.0, seed=6)
    vol = generate_array(p)
    stack = FrameStack(tuple(Frame(f, LensletGeometry(15, 15)) for f in vol))
    from paper_2310_09467_b200 import PredictorSpec
    r = pipeline.compress_stack_detailed(stack, CompressOptions(block_size=50_000,
                                                                forced=PredictorSpec(True, 1)))
    assert all(s.temporal for s in r.specs[1:])
    monkeypatch.setattr(pipeline, "DECOMPRESS_ROUND_BYTES", 2 * 256 * 160 * 2)   # two frames per round
    from paper_2310_09467_b200.codec import read_container
    h, recs, pl = read_container(r.data)
    fast = pipeline._decompress_device(h, recs, pl)
    assert fast is not None and fast == stack
    assert decompress_stack(r.data) == stack


def test_inverse_predictor_mirrors():
    """unpredict_frame / invert_predictor (reference predictors.py:101-147)
    invert predict_frame / apply_predictor exactly, every intra id, with and
    without the temporal flag."""
    from paper_2310_09467_b200 import (Frame, LensletGeometry, PredictorSpec, apply_predictor,
                                       invert_predictor, predict_frame, unpredict_frame)
    rng = np.random.default_rng(3)
    geo = LensletGeometry(6, 5)
    cur = Frame(rng.integers(0, 65536, (37, 53), dtype=np.uint16), geo)
    prev = Frame(rng.integers(0, 65536, (37, 53), dtype=np.uint16), geo)
    for i in range(13):
        assert unpredict_frame(predict_frame(cur, i), i) == cur
        for t in (False, True):
            spec = PredictorSpec(t, i)
            assert invert_predictor(apply_predictor(cur, spec, prev if t else None), spec,
                                    prev if t else None) == cur


def test_corrupt_payload_on_the_device_path_raises_like_the_reference():
    """A flipped byte in one payload of a container large enough for the
    device decoder: the block CRC check hands the container to the host path,
    which raises BlockDecodeError (blocks.py:84-92 semantics)."""
    from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry,
                                       compress_stack, decompress_stack, pipeline)
    from paper_2310_09467_b200.codec import BlockDecodeError, read_container
    p = SynthParams(512, 512, 15, 15, mode="beads", signal_amplitude=3000, noise_sigma=100,
                    photon_scale=0.05, frames=16, seed=8)
    vol = generate_array(p)
    stack = FrameStack(tuple(Frame(f, LensletGeometry(15, 15)) for f in vol))
    data = bytearray(compress_stack(stack, CompressOptions(block_size=16384)))
    h, recs, pl = read_container(bytes(data))
    assert pipeline._prefer_device_decode(h, pl, 1)
    assert decompress_stack(bytes(data)) == stack
    victim = pl[5][3]
    pos = bytes(data).find(bytes(victim))   # the payload's offset in the container
    assert pos > 0
    data[pos + len(victim) // 2] ^= 0x21
    with pytest.raises(BlockDecodeError):
        decompress_stack(bytes(data))


def test_compress_from_non_contiguous_frames():
    """pcbz_compress_frames_host takes one pointer per frame: frames that are
    strided views are made contiguous individually, and the container equals
    the one from a stacked copy."""
    from paper_2310_09467_b200 import CompressOptions, Frame, FrameStack, LensletGeometry, compress_stack
    p = SynthParams(256, 320, 15, 15, mode="smooth_lenslet", noise_sigma=10.0, photon_scale=0.05,
                    frames=3, drift=1.0, seed=12)
    vol = generate_array(p)                       # [3, 320, 256]
    wide = np.zeros((3, 320, 512), np.uint16)
    wide[:, :, ::2] = vol                         # every frame a strided view
    geo = LensletGeometry(15, 15)
    views = FrameStack(tuple(Frame(wide[i, :, ::2], geo) for i in range(3)))
    dense = FrameStack(tuple(Frame(np.ascontiguousarray(vol[i]), geo) for i in range(3)))
    opts = CompressOptions(block_size=40_000)
    assert compress_stack(views, opts) == compress_stack(dense, opts)


def test_unusual_streams_left_to_libbzip2():
    """Two concatenated streams, trailing bytes after the end-of-stream
    marker, a truncated stream and an empty stream: the device decoder takes
    only the well-formed ones (bz2.decompress semantics stay with libbzip2)."""
    rng = np.random.default_rng(21)
    a = bytes(rng.integers(0, 9, 50_000, dtype=np.uint8))
    b = bytes(rng.integers(0, 200, 30_000, dtype=np.uint8))
    pa, pb = bz2.compress(a, 9), bz2.compress(b, 9)
    cases = [(pa + pb, a + b), (pa + b"\x00\x01", a), (pa[:-7], a), (bz2.compress(b"", 9), b""), (pa, a)]
    st, got = _status([p for p, _ in cases], [len(x) for _, x in cases])
    assert list(st[:3]) == [1, 1, 1]
    assert st[3] == 0 and got[3] == b""
    assert st[4] == 0 and got[4] == a


def test_periodic_block_decoded_alone_on_host(monkeypatch):
    """A container with one exactly periodic block (a constant frame; the
    device decoder leaves it to libbzip2) still decodes on the device: only
    that payload goes through bz2.decompress, then the call is repeated
    with it supplied (pcbz_decompress_host host_streams)."""
    from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry, PredictorSpec,
                                       compress_stack, decompress_stack, pipeline)
    geo = LensletGeometry(15, 15)
    vol = generate_array(SynthParams(256, 192, 15, 15, mode="beads", signal_amplitude=3000.0,
                                     noise_sigma=20.0, photon_scale=0.05, frames=4, seed=3))
    vol[2] = 77                                    # constant frame: residual id 0 is periodic
    stack = FrameStack(tuple(Frame(f, geo) for f in vol))
    data = compress_stack(stack, CompressOptions(forced=PredictorSpec(False, 0), block_size=32768))
    calls = []
    real = bz2.decompress
    monkeypatch.setattr(pipeline.bz2, "decompress", lambda b: calls.append(len(b)) or real(b))
    monkeypatch.setattr(pipeline, "_prefer_device_decode", lambda *a: True)
    back = decompress_stack(data, workers=4)
    assert np.array_equal(back.to_array(), vol)
    nb = -(-2 * 256 * 192 // 32768)
    assert len(calls) == nb, calls                # frame 2's periodic blocks only, not the container's 4 * nb
