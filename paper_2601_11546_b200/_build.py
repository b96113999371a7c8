"""Build the sm_100a CUDA library in-tree (lib/librelserve_b200.so).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false ...

-fmad=false (and -ffp-contract=off on the host) keeps every fp64 multiply and
add separately rounded, as CPython evaluates them in the reference.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "csrc"
LIB = HERE / "lib" / "librelserve_b200.so"
SOURCES = [SRC / "engine.cu", SRC / "trace_v1.cpp"]
HEADERS = sorted(SRC.glob("*.cuh")) + [HERE.parent / "include" / "relserve.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise FileNotFoundError("nvcc not found")


def flags() -> list[str]:
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
        "-Xcompiler", "-fPIC,-ffp-contract=off",
        "-Xptxas", "-v",
        "-shared",
    ]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *flags(), "-o", str(tmp), *map(str, SOURCES)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if verbose:
        sys.stderr.write(r.stderr)
    (HERE / "lib" / "ptxas.txt").write_text(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
