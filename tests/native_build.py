"""Builds the TEST-ONLY host shim (tests/native/host_shim.cpp + the pure C++
geometry unit) with g++ so CPU tests can check the header-only device pieces
(PCG64 draws, TRF fit) and the host geometry without a GPU."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(ROOT, "paper_2303_09523_b200", "csrc")


def build_shim() -> C.CDLL:
    out = os.path.join(tempfile.gettempdir(), f"vk_host_shim_{os.getpid()}.so")
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-I", CSRC,
           os.path.join(HERE, "native", "host_shim.cpp"),
           os.path.join(CSRC, "vk_geometry.cpp"), "-o", out]
    subprocess.run(cmd, check=True)
    return C.CDLL(out)
