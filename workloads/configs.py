"""The BASELINE.json configurations as frame generators
shared by bench.py and the full-size parity tests.

  c1  one 2048x2048 bead frame (amp 3000, sigma 20, photon 0.05), pitch 15
  c2  100 independent 2048x2048 bead frames, pitch 15, three SNR levels
      (34 high: amp 20000 sigma 0 photon 0.05; 33 mid: amp 3000 sigma 100
      photon 0.05; 33 low: amp 3000 sigma 500 photon 0.01), seeds 0..99,
      13 intra candidates
  c3  2048x2048 smooth_lenslet series (amp 20000, sigma 20, photon 0.05,
      drift 1), pitch 15, temporal on (26 candidates from frame 1); "c3" is
      a 100-frame prefix of the 1000-frame series, "c3full" all of it
  c4  4096x4096 pitch-13 smooth_lenslet series, 26 candidates

Frames are bit-identical to the reference's synth.generate
(tests/golden/synth_hashes.json); series frames are made one at a time with
the reference's RNG keys, so a prefix or shard never materialises the rest.
"""
from __future__ import annotations

import multiprocessing as mpm
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass

import numpy as np

INTRA = tuple(range(13))
ALL26 = INTRA + tuple(0x80 | i for i in INTRA)
SNR_LEVELS = (  # (count, amplitude, sigma, photon) -- SURVEY.md §8(d) C2
    (34, 20000.0, 0.0, 0.05),
    (33, 3000.0, 100.0, 0.05),
    (33, 3000.0, 500.0, 0.01),
)


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    frames: int
    height: int
    width: int
    pitch: int
    codes: tuple
    temporal: bool
    series: bool      # True: one series sharded over ranks (strong), False: per-rank batch (weak)


WORKLOADS = {
    "c2": Workload("c2", "C2: 100 independent 2048x2048 uint16 bead frames, pitch 15x15, 3 SNR levels, "
                   "13 intra candidates, judge + emission", 100, 2048, 2048, 15, INTRA, False, False),
    "c1": Workload("c1", "C1: one 2048x2048 bead frame (amp 3000, sigma 20, photon 0.05), pitch 15x15, "
                   "13 intra candidates, judge + emission", 1, 2048, 2048, 15, INTRA, False, False),
    "c3": Workload("c3", "C3 prefix: 100-frame 2048x2048 smooth_lenslet series, pitch 15x15, drift 1, "
                   "temporal on (26 candidates from frame 1), frames sharded over ranks with a 1-frame halo",
                   100, 2048, 2048, 15, ALL26, True, True),
    "c3full": Workload("c3full", "C3: the full 1000-frame 2048x2048 smooth_lenslet series (8.4 GB), pitch "
                       "15x15, drift 1, temporal on (26 candidates from frame 1), frames sharded over ranks "
                       "with a 1-frame halo", 1000, 2048, 2048, 15, ALL26, True, True),
    "c4": Workload("c4", "C4: 8-frame 4096x4096 smooth_lenslet series, pitch 13x13, drift 1, temporal on "
                   "(26 candidates), frames sharded over ranks with a 1-frame halo",
                   8, 4096, 4096, 13, ALL26, True, True),
}


def c2_params():
    from .lfm_synth import SynthParams
    out, seed = [], 0
    for count, amp, sigma, photon in SNR_LEVELS:
        for _ in range(count):
            out.append(SynthParams(2048, 2048, 15, 15, mode="beads", signal_amplitude=amp,
                                   noise_sigma=sigma, photon_scale=photon, frames=1, seed=seed))
            seed += 1
    return out


def series_params(wl: Workload, frames: int | None = None):
    from .lfm_synth import SynthParams
    return SynthParams(wl.width, wl.height, wl.pitch, wl.pitch, mode="smooth_lenslet",
                       signal_amplitude=20000.0, noise_sigma=20.0, photon_scale=0.05,
                       frames=frames or wl.frames, drift=1.0, seed=0)


def _gen_one(p):
    from .lfm_synth import generate_array
    return generate_array(p)[0]


_SERIES = {}


def _gen_series_frame(t):
    from .lfm_synth import noisy_frame
    return noisy_frame(_SERIES["base"], _SERIES["params"], t)


def make_frames(wl: Workload, index, workers: int = 1) -> np.ndarray:
    """Frames `index` (a range) of the workload as a [len, H, W] uint16 array."""
    index = list(index)
    vol = np.empty((len(index), wl.height, wl.width), np.uint16)
    if wl.name == "c1":
        from .lfm_synth import SynthParams, generate_array
        vol[0] = generate_array(SynthParams(2048, 2048, 15, 15, mode="beads", signal_amplitude=3000.0,
                                            noise_sigma=20.0, photon_scale=0.05, seed=0))[0]
        return vol
    if not wl.series:
        allp = c2_params()
        params = [allp[i] for i in index]
        with ProcessPoolExecutor(max(1, workers)) as ex:
            for i, fr in enumerate(ex.map(_gen_one, params, chunksize=2)):
                vol[i] = fr
        return vol
    from .lfm_synth import scene
    p = series_params(wl)
    _SERIES["base"], _SERIES["params"] = scene(p), p   # inherited by forked workers
    with ProcessPoolExecutor(max(1, workers), mp_context=mpm.get_context("fork")) as ex:
        for i, fr in enumerate(ex.map(_gen_series_frame, index, chunksize=2)):
            vol[i] = fr
    return vol
