"""install() patches a live reference `pcbz` (imported from /root/reference in
the build container; skipped where the reference is absent, e.g. the GPU box).
CPU only: checks the bindings, no device compute."""
import os
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not present")


@pytest.fixture()
def pcbz_ref(monkeypatch):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    monkeypatch.syspath_prepend(str(REF))
    for m in [m for m in sys.modules if m == "pcbz" or m.startswith("pcbz.")]:
        monkeypatch.delitem(sys.modules, m)
    import pcbz
    import pcbz.cli  # noqa: F401  (binds select_predictor by name, cli.py:22)
    yield pcbz
    for m in [m for m in sys.modules if m == "pcbz" or m.startswith("pcbz.")]:
        sys.modules.pop(m, None)


def test_install_api_level_rebinds_every_name(pcbz_ref):
    import paper_2310_09467_b200 as b200
    from paper_2310_09467_b200 import _kernels
    orig = pcbz_ref.criterion.select_predictor
    b200.install(pcbz_ref)
    assert pcbz_ref._kernels.residual_bwt_pair_hist is _kernels.residual_bwt_pair_hist
    assert pcbz_ref._kernels.residual_image is _kernels.residual_image
    assert pcbz_ref._kernels.reconstruct_image is _kernels.reconstruct_image
    fn = pcbz_ref.criterion.select_predictor
    assert fn is not orig and fn.__wrapped_reference__ is orig
    assert pcbz_ref.pipeline.select_predictor is fn
    assert pcbz_ref.cli.select_predictor is fn
    assert pcbz_ref.select_predictor is fn


def test_install_kernel_level_keeps_numpy_entropy(pcbz_ref):
    import paper_2310_09467_b200 as b200
    orig = pcbz_ref.criterion.select_predictor
    b200.install(pcbz_ref, level="kernels")
    assert pcbz_ref.criterion.select_predictor is orig
    assert pcbz_ref._kernels.counting_bwt.__module__ == "paper_2310_09467_b200._kernels"


def test_install_validates_level(pcbz_ref):
    import paper_2310_09467_b200 as b200
    with pytest.raises(ValueError):
        b200.install(pcbz_ref, level="everything")


def test_patched_select_validates_like_reference(pcbz_ref):
    """Argument errors are raised before any device call (crit:149-154)."""
    import numpy as np
    import paper_2310_09467_b200 as b200
    b200.install(pcbz_ref)
    f = pcbz_ref.Frame(np.zeros((4, 4), np.uint16))
    with pytest.raises(ValueError):
        pcbz_ref.select_predictor(f, candidates=[])
    with pytest.raises(ValueError):
        pcbz_ref.select_predictor(f, candidates=[pcbz_ref.PredictorSpec(True, 1)])
    with pytest.raises(ValueError):
        pcbz_ref.select_predictor(f, candidates=[pcbz_ref.PredictorSpec(False, 2)] * 2)


def test_install_pipeline_level_rebinds_compress_blocks(pcbz_ref):
    """level="pipeline" also routes blocks.compress_blocks (bound by name in
    pcbz.pipeline, pipeline.py:19) to the GPU coder; streams under 1 MiB stay
    on the reference's libbzip2 path (so this runs without a GPU)."""
    import bz2
    import paper_2310_09467_b200 as b200
    orig = pcbz_ref.blocks.compress_blocks
    b200.install(pcbz_ref, level="pipeline")
    cb = pcbz_ref.blocks.compress_blocks
    assert cb is not orig and cb.__wrapped_reference__ is orig
    assert pcbz_ref.pipeline.compress_blocks is cb and pcbz_ref.compress_blocks is cb
    assert pcbz_ref.pipeline.select_predictor.__wrapped_reference__ is not None
    data = bytes(range(256)) * 100
    out = cb(data, 10000, 2)
    assert isinstance(out, pcbz_ref.blocks.CompressedBlocks)
    assert out.payloads == tuple(bz2.compress(data[i:i + 10000], 9) for i in range(0, len(data), 10000))
