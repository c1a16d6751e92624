"""GPU bzip2 back end (csrc/bzip2.cu via codec.bz2_blocks_device) against
the reference's coder call bz2.compress(chunk, 9) (blocks.py:80): byte-exact
on small and multi-block inputs, batched jobs of mixed sizes, and periodic
blocks (routed to the host libbz2)."""
import bz2
import random

import numpy as np
import pytest

import oracle
from paper_2310_09467_b200.codec import bz2_blocks_device
from workloads.lfm_synth import SynthParams, generate_array

pytestmark = pytest.mark.gpu


def _small_cases(seed, count):
    rng = random.Random(seed)
    out = [b"", b"a", b"ab", b"banana", b"aaaa", b"aaaaa", b"a" * 255, b"a" * 256, b"a" * 260,
           bytes(range(256)), b"ab" * 3 + b"c"]
    for _ in range(count):
        n = rng.choice([1, 2, 3, 5, 9, 17, 100, 700, 2000, 20000])
        alph = rng.choice([2, 3, 16, 256])
        s = bytearray()
        while len(s) < n:
            s += bytes([rng.randrange(alph)]) * (rng.randint(1, 300) if rng.random() < 0.1 else rng.randint(1, 6))
        out.append(bytes(s[:n]))
    return out


def test_small_inputs_one_batch():
    cases = _small_cases(11, 200)
    got = bz2_blocks_device(cases)
    for c, g in zip(cases, got):
        assert g == bz2.compress(c, 9), (len(c), c[:24])


def test_multiblock_streams():
    img = generate_array(SynthParams(2048, 2048, 15, 15, mode="beads", signal_amplitude=3000,
                                     noise_sigma=100, photon_scale=0.05, seed=3))[0]
    st = oracle.emit_stream(img, None, 4, 15, 15)
    rng = np.random.default_rng(0)
    cases = [st[:4 << 20], st[4 << 20:], rng.integers(0, 256, 2_000_000, dtype=np.uint8).tobytes(),
             (rng.integers(0, 4, 1_900_000, dtype=np.uint8) * 0).tobytes(),           # zeros: periodic
             bytes(rng.integers(0, 256, 997, dtype=np.uint8)) * 1200]                  # periodic, long period
    got = bz2_blocks_device(cases)
    for c, g in zip(cases, got):
        assert g == bz2.compress(c, 9), len(c)


def test_residual_streams_batch_like_pipeline():
    """The pipeline's use: 4 MiB blocks of residual streams of many frames."""
    vol = generate_array(SynthParams(1024, 1024, 15, 15, mode="smooth_lenslet", noise_sigma=20.0,
                                     photon_scale=0.05, frames=4, drift=1.0, seed=1))
    chunks = []
    for f in range(4):
        s = oracle.emit_stream(vol[f], vol[f - 1] if f else None, 12 | (0x80 if f else 0), 15, 15)
        chunks += [s[i:i + 700_000] for i in range(0, len(s), 700_000)]
    got = bz2_blocks_device(chunks)
    for c, g in zip(chunks, got):
        assert g == bz2.compress(c, 9)
