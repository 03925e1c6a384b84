"""Build libcurvigpu.so in-tree with nvcc for sm_100a.

    python -m paper_2604_11558_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libcurvigpu.so"
SOURCES = [CSRC / "plan.cu", CSRC / "setup.cu", CSRC / "rng.cpp"]
HEADERS = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "curvigpu.h"]
DEPS = SOURCES + HEADERS
OBJ_DIR = PKG / "build"   # git-ignored objects, one per translation unit

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    cmd = [nvcc(), *NVCC_FLAGS, f"-I{ROOT / 'include'}", "-c", "-o", str(obj), str(src)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit for sm_100a (in parallel; an object is
    reused only when it is newer than its source and every header) and link
    libcurvigpu.so.  ``force`` recompiles everything."""
    from concurrent.futures import ThreadPoolExecutor

    newest_hdr = max(p.stat().st_mtime for p in HEADERS)
    OBJ_DIR.mkdir(exist_ok=True)
    objs, todo = [], []
    for src in SOURCES:
        obj = OBJ_DIR / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_hdr):
            todo.append((src, obj))
    if not todo and OUT.exists() and OUT.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return OUT
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        for fut in [pool.submit(_compile, src, obj, verbose) for src, obj in todo]:
            fut.result()
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
