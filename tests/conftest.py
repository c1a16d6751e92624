import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libpcbz_b200.so")
    config.addinivalue_line("markers", "slow: several seconds of CPU work")


def gpu_available() -> bool:
    try:
        from paper_2310_09467_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # -m gpu runs on the B200 box: a missing device or library there must FAIL
    # (no silent skip, no CPU fallback), so nothing is skipped here.
    pass


@pytest.fixture(scope="session")
def golden_small():
    meta = json.loads((GOLDEN / "small_cases.json").read_text())
    arrays = np.load(GOLDEN / "small_cases.npz")
    return meta, arrays


@pytest.fixture(scope="session")
def golden_kats():
    return json.loads((GOLDEN / "kats.json").read_text())


@pytest.fixture(scope="session")
def golden_medium():
    return json.loads((GOLDEN / "medium_cases.json").read_text())


@pytest.fixture(scope="session")
def golden_synth():
    return json.loads((GOLDEN / "synth_hashes.json").read_text())


@pytest.fixture(scope="session")
def golden_c1():
    return json.loads((GOLDEN / "c1_2048.json").read_text())


def log2_fingerprint() -> str:
    """sha256 of this host's np.log2 over the entropy probabilities of a
    2048x2048 frame (p = c / (2*2048*2048 - 1), c = 1..65535) and 65536
    random doubles in (0, 1].  numpy picks its log2 implementation by CPU
    features at run time (not correctly rounded on AVX-512 hosts), so the
    reference's entropies are bit-reproducible only on hosts with the same
    fingerprint as the one that generated the goldens."""
    N = 2 * 2048 * 2048 - 1
    p = np.arange(1, 65536, dtype=np.int64) / float(N)
    q = 1.0 - np.random.default_rng(0).random(65536)
    return sha(np.concatenate([np.log2(p), np.log2(q)]))


@pytest.fixture(scope="session")
def same_log2_as_golden() -> bool:
    want = json.loads((GOLDEN / "log2_fingerprint.json").read_text())["sha256"]
    return log2_fingerprint() == want


def golden_hist(arrays, name, fi, code):
    h = np.zeros(65536, np.int64)
    h[arrays[f"{name}/f{fi}/c{code}/bins"]] = arrays[f"{name}/f{fi}/c{code}/counts"]
    return h


def sha(b) -> str:
    import hashlib
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()
