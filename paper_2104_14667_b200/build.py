"""Build libfloodstream.so in-tree with nvcc for sm_100a.

The library is the product path of this package: every per-pixel and pairwise kernel
of the flood-ensemble overlap path runs from it.  It is built in the source tree
(``paper_2104_14667_b200/_lib/``) so the artefact travels with the repository snapshot;
there is no JIT cache and no CPU fallback.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libfloodstream.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["fs_kernels.cu", "fs_gram_tc.cu", "fs_recompute_f4.cu", "fs_capi.cu", "fs_pipeline.cu"]
HEADERS = ["fs_common.cuh", "fs_internal.h", "fs_bitslice.cuh", "fs_tcgen05.cuh"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfloodstream")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE / "floodstream.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          extra: list[str] | None = None) -> Path:
    """Build the library (default: in-tree, when stale).  ``out`` / ``extra``: a probe
    build with extra nvcc flags at another path (timing experiments only)."""
    target = Path(out) if out is not None else LIB
    if out is None and not force and not _stale():
        return LIB
    target.parent.mkdir(parents=True, exist_ok=True)
    tmp = target.with_suffix(".so.tmp")
    cmd = [
        nvcc(),
        *ARCH_FLAGS,
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-shared",
        "-Xcompiler",
        "-fPIC,-ffp-contract=off,-O3",
        "-I",
        str(INCLUDE),
        "-I",
        str(CSRC),
        *(["-Xptxas", "-v"] if verbose else []),
        # experiment knobs (e.g. -DFS_EXP_BATCH=1); never set for the shipped build
        *os.environ.get("FS_NVCC_EXTRA", "").split(),
        *(extra or []),
        *[str(CSRC / s) for s in SOURCES],
        "-o",
        str(tmp),
    ]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libfloodstream (see stderr)")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
