"""In-tree build of libqgpu.so (sm_100a) with nvcc.

The shared library is written to ``paper_1802_08032_b200/_lib/libqgpu.so``
(git-ignored, shipped to the GPU box with the gpurun snapshot). Objects are
rebuilt only when a source or header is newer than them.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = PKG / "_lib" / "obj"
LIB = PKG / "_lib" / "libqgpu.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3", "-std=c++20", "-lineinfo", "--fmad=false",
    "-Xcompiler", "-fPIC,-O3,-ffp-contract=off",
    # one brx.idx jump table per op switch instead of NVVM's binary
    # search tree of compares and branches (tile_pass.cu: step)
    "-Xcicc", "-jump-table-density=1",
    f"-I{INCLUDE}", f"-I{CSRC}",
]
SOURCES = ["kernels.cu", "tile_pass.cu", "runtime.cpp", "api.cpp", "transport.cpp", "memory_plan.cpp", "swap_plan.cpp"]


def _headers() -> list[Path]:
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: str, verbose: bool) -> Path:
    s = CSRC / src
    o = OBJ / (s.stem + ".o")
    if _stale(o, [s, *_headers()]):
        cmd = [NVCC, *ARCH, *COMMON, "-x", "cu" if src.endswith(".cu") else "c++", "-c", str(s), "-o", str(o)]
        if src.endswith(".cu"):
            cmd.insert(1, "-Xptxas=-v") if verbose else None
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    return o


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
