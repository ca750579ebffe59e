"""Build libb200tally.so in-tree with nvcc for sm_100a.

--fmad=false is part of the arithmetic contract (bit-exact walks, see
csrc/geometry.cuh); never add --use_fast_math.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc" / "b200tally.cu"
DEPS = [SRC, *sorted((PKG / "csrc").glob("*.cuh")), PKG / "csrc" / "glibc_tables.inc",
        ROOT / "include" / "b200tally.h"]
LIB = PKG / "libb200tally.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "--fmad=false", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(d.stat().st_mtime > t for d in DEPS)


TABLES = PKG / "csrc" / "glibc_tables.inc"


def build(force: bool = False, verbose: bool = False) -> Path:
    # the host libm's log / sin / cos tables for the transport (not committed;
    # rewritten only when they change, so an unchanged build stays up to date)
    try:
        from . import glibc_tables
    except ImportError:  # run as a script
        sys.path.insert(0, str(PKG))
        import glibc_tables
    glibc_tables.generate(TABLES)
    if not force and not needs_build():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-o", str(LIB), str(SRC)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
