"""lfm_synth must reproduce the reference generator bit for bit (hashes made by
the reference, tests/golden/synth_hashes.json).  CPU only."""
import pytest

from conftest import sha
from workloads.lfm_synth import SynthParams, generate_array

FAST = ["small_smooth", "small_beads"]
SLOW = ["c1_beads_2048_p15", "c2_high_seed1", "c2_mid_seed40", "c2_low_seed80", "c3_series_prefix3"]


@pytest.mark.parametrize("name", FAST)
def test_small(golden_synth, name):
    g = golden_synth[name]
    vol = generate_array(SynthParams(**g["params"]))
    assert list(vol.shape) == g["shape"]
    assert sha(vol) == g["sha"]


@pytest.mark.slow
@pytest.mark.parametrize("name", SLOW)
def test_full_size(golden_synth, name):
    g = golden_synth[name]
    vol = generate_array(SynthParams(**g["params"]))
    assert sha(vol) == g["sha"]


def test_params_validation():
    with pytest.raises(ValueError):
        SynthParams(0, 4)
    with pytest.raises(ValueError):
        SynthParams(4, 4, mode="vessels")
    with pytest.raises(ValueError):
        SynthParams(4, 4, signal_amplitude=65000.0, noise_sigma=200.0)
