"""Build libsqf2k_b200.so in-tree: hand-written CUDA for sm_100a (B200).

    python -m paper_2411_01964_b200.build [--force] [--verbose]

nvcc cross-compiles without a GPU; the .so lands next to this file so it
travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libsqf2k_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["context.cu", "primes.cu", "tile.cu", "verify.cu", "scan.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-diag-suppress", "186"]
OBJ = PKG / "_obj"


def _inputs() -> list[Path]:
    return [CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "sqf2k_b200.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _inputs())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Each source compiles to an object in parallel (no cross-file device
    code: relocatable device code is not needed), then one host link."""
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    OBJ.mkdir(exist_ok=True)
    extra = os.environ.get("SQF2K_NVCC_EXTRA", "").split()  # build options, e.g. -DSQF2K_...=1
    tag = f"{os.getpid()}"

    def compile_one(src: str) -> Path:
        obj = OBJ / f"{Path(src).stem}.{tag}.o"
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", str(INCLUDE), "-c", "-o", str(obj),
               str(CSRC / src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB.with_name(f".{LIB.name}.{tag}.tmp")
    try:
        subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp),
                        *map(str, objs)], check=True)
    finally:
        for o in objs:
            o.unlink(missing_ok=True)
    os.replace(tmp, LIB)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
