"""The C ABI from plain C: the header and the
example caller compile as C99 against include/volkrig_b200.h and link against
the built library (CPU), and the program runs on the device (GPU)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "c_abi_example.c")
LIBDIR = os.path.join(ROOT, "paper_2303_09523_b200", "_native")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    if not os.path.exists(os.path.join(LIBDIR, "libvolkrig_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path / "c_abi_example")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-o", exe, SRC,
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           "-L", LIBDIR, "-lvolkrig_b200", "-L", f"{CUDA}/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_and_caller_compile_as_c99(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_caller_runs_on_device(cuda, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert "fast_path=1" in r.stdout and "known_exact=1" in r.stdout and "failed_part=-1" in r.stdout
