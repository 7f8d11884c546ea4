"""CPU: the C-ABI library loads without a GPU and exports exactly the entry
points include/volkrig_b200.h declares; the Python layer binds them all and
fails loudly (no fallback) when no CUDA device is present."""

import os
import re

import pytest

from paper_2303_09523_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "volkrig_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ("vk_plan_create", "vk_plan_execute", "vk_plan_finish", "vk_fit_variogram_samples",
              "vk_sample_pairs", "vk_grid_scan", "vk_gather_planes"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_python_binding_covers_header():
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_status_strings_and_version():
    lib = _lib.load()
    assert lib.vk_abi_version() == 1
    assert lib.vk_status_string(0) == b"ok"
    assert lib.vk_status_string(3) == b"singular kriging system"


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np
    from paper_2303_09523_b200 import DeviceError, VariogramModel, VolumeGrid, fill_missing
    d = np.zeros((3, 4, 4), np.float32)
    d[1] = np.nan
    with pytest.raises(DeviceError):
        fill_missing(VolumeGrid(d), VariogramModel("exponential", 0, 1, 1))


def test_error_mapping():
    from paper_2303_09523_b200 import errors as E
    with pytest.raises(E.SingularSystem):
        E.raise_for_status(_lib.VK_E_SINGULAR_SYSTEM)
    with pytest.raises(E.NoKnownNeighbors):
        E.raise_for_status(_lib.VK_E_NO_KNOWN_NEIGHBORS)
    with pytest.raises(ValueError):
        E.raise_for_status(_lib.VK_E_INVALID_GRID)
    assert E.exit_code_for(E.SingularSystem()) == 7
