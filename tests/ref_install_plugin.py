"""pytest plugin (-p ref_install_plugin) used by tests/test_reference_suite.py:
before the reference's own test modules are collected -- they bind
select_predictor and the kernels by name at import -- import the reference
package from baseline/_ref and patch it with paper_2310_09467_b200.install()
at PCBZ_INSTALL_LEVEL ("api" / "kernels"; "none" = unpatched control run)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STATE = {}


def pytest_configure(config):
    level = os.environ.get("PCBZ_INSTALL_LEVEL", "api")
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    sys.path.insert(0, str(ROOT))
    import pcbz
    import pcbz.cli  # noqa: F401  (binds select_predictor by name, cli.py:22)
    assert Path(pcbz.__file__).resolve().is_relative_to(ROOT / "baseline" / "_ref"), pcbz.__file__
    if level != "none":
        import paper_2310_09467_b200 as b200
        b200.install(pcbz, level=level)
        assert pcbz._kernels.residual_bwt_pair_hist.__module__ == "paper_2310_09467_b200._kernels"
    STATE["level"] = level


def pytest_report_header(config):
    return f"reference pcbz from baseline/_ref, paper_2310_09467_b200.install level={STATE.get('level')}"
