"""Build experimental variants (fast path for pitch 15 only, the C2 bench pitch) of libpcbz_b200.so side by side for A/B runs
(select one at run time with PCBZ_LIB=<path>)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2310_09467_b200 import build_native  # noqa: E402

VARIANTS = {
    "base": (),
    "incptr": ("PCBZ_INCPTR=1",),
    "defer": ("PCBZ_DEFER=1",),
    "incptr_defer": ("PCBZ_INCPTR=1", "PCBZ_DEFER=1"),
    "inline": ("PCBZ_LANE_INLINE=1",),
    "incptr_inline": ("PCBZ_INCPTR=1", "PCBZ_LANE_INLINE=1"),
    "half_lsb": ("PCBZ_HALF_MSB=0",),
    "pf4": ("PCBZ_PREFETCH=4",),
    "pf8": ("PCBZ_PREFETCH=8",),
    "pf16": ("PCBZ_PREFETCH=16",),
    "pf32": ("PCBZ_PREFETCH=32",),
    "evict_last": ("PCBZ_LDG_HINT=1",),
    "emit_chunks": ("PCBZ_EMIT_RUNS=0",),
    "emit_run2": ("PCBZ_EMIT_RUN=2",),
    "emit_run8": ("PCBZ_EMIT_RUN=8",),
    "emit_run16": ("PCBZ_EMIT_RUN=16",),
    "emit_run1": ("PCBZ_EMIT_RUN=1",),
    "emit_run1_m8": ("PCBZ_EMIT_RUN=1", "PCBZ_EMIT_MINB=8"),
    "emit_run2_m6": ("PCBZ_EMIT_RUN=2", "PCBZ_EMIT_MINB=6"),
    "emit_run2_m8": ("PCBZ_EMIT_RUN=2", "PCBZ_EMIT_MINB=8"),
    "emit_run4_m6": ("PCBZ_EMIT_RUN=4", "PCBZ_EMIT_MINB=6"),
    "trace5": ("PCBZ_TRACE_WORDS=5",),
    "trace9": ("PCBZ_TRACE_WORDS=9",),
    "fin192": ("PCBZ_FINALIZE_THREADS=192",),
    "fin384": ("PCBZ_FINALIZE_THREADS=384",),
    "fin512": ("PCBZ_FINALIZE_THREADS=512",),
    "fin768": ("PCBZ_FINALIZE_THREADS=768",),
}

def build_from_git(rev: str, name: str):
    """Baseline for an A/B run: the library as of git revision `rev`."""
    import subprocess
    import tarfile
    import tempfile
    tmp = Path(tempfile.mkdtemp(prefix="pcbz_ab_"))
    data = subprocess.run(["git", "-C", str(ROOT), "archive", rev, "paper_2310_09467_b200/csrc",
                           "include"], check=True, capture_output=True).stdout
    import io
    tarfile.open(fileobj=io.BytesIO(data)).extractall(tmp)
    out = ROOT / "paper_2310_09467_b200" / "_native" / "variants" / name
    print(name, build_native.build_library(force=True, out_dir=out, pitches={15}, src_root=tmp),
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) == 4 and sys.argv[1] == "--git":   # --git REV NAME
        build_from_git(sys.argv[2], sys.argv[3])
        sys.exit(0)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        out = ROOT / "paper_2310_09467_b200" / "_native" / "variants" / n
        # VARIANT_PITCHES=13,15: fast-path pitches to instantiate (others abort if selected)
        import os
        pitches = {int(x) for x in os.environ.get("VARIANT_PITCHES", "15").split(",")}
        print(n, build_native.build_library(force=True, defines=VARIANTS[n], out_dir=out, pitches=pitches),
              flush=True)
