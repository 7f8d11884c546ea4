"""Builds the in-tree CUDA library ``_native/libvolkrig_b200.so`` for sm_100a.

The library is a plain C ABI (``include/volkrig_b200.h``); it is compiled
with nvcc directly (no torch extension), so it carries no torch types and can
be bound from any FFI.  Where the reference's arithmetic must be reproduced
bit for bit (lags, half squared differences, bin edges and centres) the
kernels use explicit round-to-nearest intrinsics, so FMA contraction stays on
everywhere else.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_native"
LIB = OUT_DIR / "libvolkrig_b200.so"
INCLUDE = PKG.parent / "include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

UNITS = {
    "vk_api.cu": [],
    # ptxas -O1: the fit kernel is a 31 k-instruction serial FP64 chain that
    # waits on instruction fetches a fifth of the time; the default level's
    # scheduling buys it nothing (C4 fit 1.479 -> 1.449 ms, C2 1.058 -> 1.047;
    # the unit's bandwidth kernels measure the same; bits unchanged -- FMA
    # contraction is decided before ptxas)
    "vk_variogram.cu": ["-Xptxas", "-O1"],
    "vk_npstats.cu": [],
    "vk_solve.cu": [],
    "vk_predict.cu": [],
    "vk_predict_fixed.cu": [],
    "vk_generic.cu": [],
    "vk_volio.cu": [],
    "vk_geometry.cpp": [],
    "vk_comm.cpp": [],
    "vk_hostio.cpp": [],
}


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    deps = _deps()
    for unit, extra in UNITS.items():
        src = CSRC / unit
        obj = OUT_DIR / (unit + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src] + deps + [Path(__file__)]):
            continue
        exp = os.environ.get("VK_NVCC_EXTRA", "").split()    # tuning experiments only
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", str(INCLUDE), "-I", str(CSRC), *extra, *exp, "-c", str(src),
               "-o", str(obj)]
        if unit.endswith(".cpp") and unit not in ("vk_comm.cpp", "vk_hostio.cpp"):
            cmd.insert(1, "-x")
            cmd.insert(2, "cu")
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs),
               "-cudart", "static", "-ldl"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
