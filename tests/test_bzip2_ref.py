"""Pins oracle/bzip2_ref.py (the restated libbzip2 1.0.8 level-9 compressor,
oracle of the GPU block coder) byte-for-byte against bz2.compress(x, 9),
the call the reference makes (blocks.py:80).  Blocks whose rotations tie
(exactly periodic blocks) are flagged, not restated: libbz2 orders equal
rotations by its quicksort refinements, so those inputs go to host bzip2."""
import bz2
import random

import numpy as np
import pytest

import bzip2_ref as R
import oracle
from workloads.lfm_synth import SynthParams, generate_array


def _cases(seed, count):
    rng = random.Random(seed)
    out = [b"", b"a", b"ab", b"banana", b"aaaa", b"aaaaa", b"a" * 255, b"a" * 256, b"a" * 260,
           b"ab" * 3 + b"c", bytes(range(256))]
    for _ in range(count):
        n = rng.choice([1, 2, 3, 5, 9, 17, 100, 700, 2000])
        alph = rng.choice([2, 3, 16, 256])
        s = bytearray()
        while len(s) < n:
            s += bytes([rng.randrange(alph)]) * (rng.randint(1, 300) if rng.random() < 0.1 else rng.randint(1, 6))
        out.append(bytes(s[:n]))
    return out


def test_restated_compressor_matches_libbz2():
    ties = 0
    for c in _cases(7, 150):
        trace = []
        got = R.compress(c, trace)
        if any(t["tie"] for t in trace):
            ties += 1
            continue
        assert got == bz2.compress(c, 9), c[:32]
    assert ties < 60


def test_periodic_blocks_are_flagged():
    for s in (b"ab" * 50, b"\x00\x00", bytes(range(256)) * 3, b"xyz" * 1000):
        trace = []
        R.compress(s, trace)
        assert any(t["tie"] for t in trace)


def test_multiblock_residual_stream():
    """Two level-9 blocks (899,981-byte RLE1 boundary, a pending run carried
    into the next block) of a real residual stream."""
    img = generate_array(SynthParams(1024, 1024, 15, 15, mode="beads", signal_amplitude=3000,
                                     noise_sigma=100, photon_scale=0.05, seed=3))[0]
    st = oracle.emit_stream(img, None, 4, 15, 15)[:1_200_000]
    trace = []
    assert R.compress(st, trace) == bz2.compress(st, 9)
    assert [t["n"] for t in trace][0] >= R.BLOCK_MAX and len(trace) == 2


def test_code_lengths_respect_max_len():
    rng = np.random.default_rng(0)
    freq = list((rng.pareto(0.5, 258) * 1000).astype(int))      # very skewed: forces rescaling
    lens = R.make_code_lengths(freq, 258, 17)
    assert max(lens) <= 17 and sum(2.0 ** -l for l in lens) <= 1.0 + 1e-12
