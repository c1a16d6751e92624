"""Streaming compression (pipeline.compress_stream + codec.ContainerWriter)
on CPU: the oracle stands in for the device judge; the container must equal
the single-shot reference restatement byte for byte, for seekable and
non-seekable outputs and any chunking."""
import io

import numpy as np
import pytest

import oracle
from conftest import sha
from paper_2310_09467_b200 import CompressOptions, PredictorSpec
from paper_2310_09467_b200.codec import ContainerWriter, write_container, CompressedBlocks, BlockPlan
from paper_2310_09467_b200.core import LensletGeometry
from workloads.lfm_synth import SynthParams, generate_array
from paper_2310_09467_b200.pipeline import compress_stream


def oracle_judge(frames, halo, geo, codes, temporal):
    F = frames.shape[0]
    ent = np.full((F, len(codes)), np.nan)
    sel = np.zeros(F, np.uint8)
    streams, prev = [], halo
    for f in range(F):
        cands = [c for c in codes if (prev is not None and temporal) or not c & 0x80]
        entries, best, _ = oracle.select_predictor(frames[f], prev if temporal else None, cands,
                                                   geo.pitch_x, geo.pitch_y)
        for c, e in entries:
            ent[f, codes.index(c)] = e
        sel[f] = best
        streams.append(np.frombuffer(oracle.emit_stream(frames[f], prev, best, geo.pitch_x,
                                                        geo.pitch_y), np.uint8))
        prev = frames[f]
    return ent, sel, np.stack(streams)


class _NoSeek(io.RawIOBase):
    def __init__(self):
        self.buf = bytearray()

    def writable(self):
        return True

    def seekable(self):
        return False

    def write(self, b):
        self.buf += bytes(b)
        return len(b)


@pytest.fixture(scope="module")
def series():
    return generate_array(SynthParams(40, 33, 6, 5, mode="smooth_lenslet", noise_sigma=30.0,
                                      photon_scale=0.05, frames=7, drift=0.5, seed=3))


@pytest.mark.parametrize("chunk,announce,seekable", [(1, True, True), (3, True, True),
                                                     (3, False, True), (2, True, False),
                                                     (7, False, False), (16, True, True)])
def test_stream_equals_single_shot(series, chunk, announce, seekable):
    out = io.BytesIO() if seekable else _NoSeek()
    res = compress_stream(iter(list(series)), LensletGeometry(6, 5), out,
                          CompressOptions(workers=3, block_size=700),
                          nframes=len(series) if announce else None, chunk_frames=chunk,
                          max_inflight_chunks=2, judge_fn=oracle_judge)
    got = out.getvalue() if seekable else bytes(out.buf)
    want, _ = oracle.compress_stack(series, 6, 5, block_size=700)
    assert sha(got) == sha(want)
    assert res.frames == len(series) and res.container_bytes == len(got)


def test_stream_temporal_off(series):
    geo = LensletGeometry(6, 5)
    out = io.BytesIO()
    compress_stream(series, geo, out, CompressOptions(temporal=False), chunk_frames=2,
                    judge_fn=oracle_judge)
    want, _ = oracle.compress_stack(series, 6, 5, temporal=False)
    assert sha(out.getvalue()) == sha(want)


def test_writer_validation():
    w = ContainerWriter(io.BytesIO(), 4, 4, 1, 1, 16, nframes=2)
    with pytest.raises(ValueError):
        w.add_frame(PredictorSpec(True, 1), [b"x", b"y"])        # temporal frame 0
    with pytest.raises(ValueError):
        w.add_frame(PredictorSpec(False, 1), [b"x"])              # wrong block count
    w.add_frame(PredictorSpec(False, 1), [b"x", b"y"])
    with pytest.raises(ValueError):
        w.close()                                                  # 1 of 2 announced frames
    with pytest.raises(ValueError):
        compress_stream(iter([]), LensletGeometry(1, 1), io.BytesIO(), judge_fn=oracle_judge)


def test_writer_matches_write_container():
    specs = [PredictorSpec(False, 3), PredictorSpec(True, 0), PredictorSpec(True, 12)]
    payloads = [(b"ab", b"c"), (b"", b"defg"), (b"h", b"ij")]
    frames = [(s, CompressedBlocks(BlockPlan(16, 2), p)) for s, p in zip(specs, payloads)]
    want = write_container(4, 4, 2, 3, 16, frames)
    for n in (3, None):
        buf = io.BytesIO()
        w = ContainerWriter(buf, 4, 4, 2, 3, 16, nframes=n)
        for s, p in zip(specs, payloads):
            w.add_frame(s, list(p))
        assert w.close() == len(want)
        assert buf.getvalue() == want
