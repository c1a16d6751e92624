"""Short runs of the randomised stress tools (tools/stress_*.py) as GPU
tests: random shapes, pitches, value kinds, segment overrides, band counts,
garbage outside a band's rows, options and coders, each case checked
against the oracle (and the whole-frame judge for bands).  The long runs
are logged under profiles/r02_stress_*.log."""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(tool, *args, monkeypatch=None):
    sys.path[:0] = [str(ROOT / "tools")]
    try:
        mod = __import__(tool)
        monkeypatch.setattr(sys, "argv", [tool, *map(str, args)])
        return mod.main()
    finally:
        sys.path.remove(str(ROOT / "tools"))


@pytest.mark.gpu
def test_stress_judge(monkeypatch, capsys):
    assert _run("stress_parity", 120, 31, monkeypatch=monkeypatch) == 0, capsys.readouterr().out


@pytest.mark.gpu
def test_stress_bands(monkeypatch, capsys):
    assert _run("stress_bands", 150, 32, monkeypatch=monkeypatch) == 0, capsys.readouterr().out


@pytest.mark.gpu
def test_stress_roundtrip(monkeypatch, capsys):
    assert _run("stress_roundtrip", 40, 33, monkeypatch=monkeypatch) == 0, capsys.readouterr().out
