"""Build experimental variants (fast path for pitch 15 only, the C2 bench pitch) of libpcbz_b200.so side by side for A/B runs
(select one at run time with PCBZ_LIB=<path>)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2310_09467_b200 import build_native  # noqa: E402

VARIANTS = {
    "half_lsb": ("PCBZ_HALF_MSB=0",),
    "half_msb": ("PCBZ_HALF_MSB=1",),
    "half_lsb_noswz": ("PCBZ_HALF_MSB=0", "PCBZ_SWIZZLE=0"),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        out = ROOT / "paper_2310_09467_b200" / "_native" / "variants" / n
        print(n, build_native.build_library(force=True, defines=VARIANTS[n], out_dir=out, pitches={15}), flush=True)
