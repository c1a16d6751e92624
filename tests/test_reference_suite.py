"""The reference's own test suite (pcbz/tests, staged by
tools/install_reference.sh into baseline/_ref/pcbz_tests next to the
unmodified reference package) run with the B200 path patched in through
paper_2310_09467_b200.install(): level="api" (device
select_predictor, entropies from this host's numpy terms) and
level="kernels" (device kernels under the reference's own numpy
entropy2d).  Fails -- does not skip -- when the reference is not staged."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref" / "pcbz_tests"

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("level", ["api", "kernels"])
def test_reference_suite_under_install(level, tmp_path):
    assert (SUITE / "test_criterion.py").exists(), \
        "reference suite not staged: run tools/install_reference.sh (baseline/_ref travels with gpurun)"
    env = dict(os.environ, PCBZ_INSTALL_LEVEL=level, NUMBA_CACHE_DIR=str(tmp_path / "numba"),
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), str(ROOT / "baseline" / "_ref"), str(ROOT)]))
    r = subprocess.run([sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "ref_install_plugin",
                        "-p", "no:cacheprovider", "-x", "-n", "8", "--rootdir", str(SUITE)],
                       cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-30:])
    print(tail)
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail
