"""Build libpcbz_b200.so (sm_100a) in-tree with nvcc, and the C oracle.

Used by __graft_entry__.build() and by `python -m paper_2310_09467_b200.build_native`.
The shared library lands in paper_2310_09467_b200/_native/ so it travels with
the repository snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
The histogram kernel is instantiated once per fast-path pitch (judge_px.cu
with -DPCBZ_PX=0..16); those translation units compile in parallel.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_native"
LIB = OUT_DIR / "libpcbz_b200.so"
MAX_FAST_PITCH = 16

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libpcbz_b200.so")


def _units(pitches=None):
    """(source, extra flags, object name) of every translation unit; pitches
    not in `pitches` (None = all) get an empty stub."""
    units = [("judge.cu", [], "judge.o"), ("aux_kernels.cu", [], "aux_kernels.o"),
             ("capi.cu", [], "capi.o"), ("bzip2.cu", [], "bzip2.o"),
             ("bunzip2.cu", [], "bunzip2.o")]
    for px in range(MAX_FAST_PITCH + 1):
        stub = pitches is not None and px not in pitches and px != 0
        units.append(("judge_px.cu", [f"-DPCBZ_PX={px}"] + (["-DPCBZ_STUB=1"] if stub else []),
                      f"judge_px{px}.o"))
    return units


def _deps():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "pcbz_b200.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False, jobs: int | None = None,
                  defines: tuple = (), out_dir: Path | None = None, pitches=None,
                  src_root: Path | None = None) -> Path:
    """Compile and link libpcbz_b200.so.  `defines` / `out_dir` build an
    experimental variant (e.g. ("PCBZ_SWIZZLE=0",)) into its own directory;
    `src_root` builds from another tree holding paper_2310_09467_b200/csrc and
    include/ (an A/B baseline exported from git, tools/build_variants.py);
    _lib.load() picks a variant up through the PCBZ_LIB environment variable."""
    csrc = Path(src_root) / "paper_2310_09467_b200" / "csrc" if src_root else CSRC
    inc = Path(src_root) / "include" if src_root else ROOT / "include"
    out = Path(out_dir) if out_dir else OUT_DIR
    lib = out / LIB.name
    if not force and not _stale(lib, _deps()):
        return lib
    out.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    dflags = [f"-D{d}" for d in defines]

    def compile_one(unit):
        src, extra, obj = unit
        cmd = [nvcc, *NVCC_FLAGS, *dflags, *extra, "-I", str(inc), "-c",
               str(csrc / src), "-o", str(out / obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} {extra}:\n{r.stdout}\n{r.stderr}")
        return f"== {src} {' '.join(extra)}\n{r.stdout}{r.stderr}"

    units = _units(pitches)
    with ThreadPoolExecutor(jobs or max(1, os.cpu_count() or 1)) as pool:
        logs = list(pool.map(compile_one, units))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *[str(out / u[2]) for u in units],
           "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    (out / "ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


def build_oracle() -> Path | None:
    """Compile the C oracle (test infrastructure) with its Makefile."""
    mk = ROOT / "oracle" / "Makefile"
    if not mk.exists():
        return None
    r = subprocess.run(["make", "-s", "-C", str(mk.parent)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return mk.parent / "build" / "liboracle.so"


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_oracle())
