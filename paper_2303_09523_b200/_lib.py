"""ctypes binding of the in-tree C ABI (``include/volkrig_b200.h``).

The library is loaded from ``paper_2303_09523_b200/_native``.  There is no
fallback: if it is missing or fails to load, every compute entry point raises
``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_native" / "libvolkrig_b200.so"

VK_OK = 0
VK_E_INVALID_ARGUMENT = 1
VK_E_NO_KNOWN_NEIGHBORS = 2
VK_E_SINGULAR_SYSTEM = 3
VK_E_INSUFFICIENT_SAMPLES = 4
VK_E_DEGENERATE_LAGS = 5
VK_E_UNSUPPORTED = 6
VK_E_CUDA = 7
VK_E_INVALID_GRID = 8
VK_E_FIT_FAILED = 9

KIND_IDS = {"exponential": 0, "gaussian": 1, "spherical": 2}
DRIFT_IDS = {"linear": 0, "constant": 1}
ACCUM_IDS = {"fp64": 0, "fp32": 1, "fixed": 2}
FLAG_FORCE_GENERIC = 1
FLAG_REDRAW_PAIRS = 2
FLAG_OVERLAP = 4
FLAG_SERIAL = 8
N_STAGES = 6
STAGES = ("stats", "pairs", "bins", "fit", "solve", "predict")


class NativeLibraryMissing(RuntimeError):
    pass


class PlanDesc(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("depth", C.c_int32),
                ("n_known", C.c_int32), ("known_z", C.POINTER(C.c_int32)),
                ("n_subparts", C.c_int32), ("kind", C.c_int32), ("drift", C.c_int32),
                ("accum", C.c_int32), ("n_bins", C.c_int32), ("max_pairs", C.c_int64),
                ("seed", C.c_uint64), ("fit_variogram", C.c_int32), ("flags", C.c_int32),
                ("part_len", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("fast_path", C.c_int32), ("gap_planes", C.c_int32),
                ("n_patterns", C.c_int32), ("n_kinds", C.c_int32),
                ("n_systems", C.c_int32), ("n_missing_planes", C.c_int32),
                ("n_pair_classes", C.c_int32), ("kernels_per_execute", C.c_int32),
                ("interpolated_voxels", C.c_int64)]


# name -> (restype, argtypes); every symbol the header declares
SIGNATURES = {
    "vk_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]),
    "vk_plan_destroy": (None, [C.c_void_p]),
    "vk_plan_execute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "vk_plan_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32),
                                 C.c_void_p, C.c_void_p]),
    "vk_plan_get_info": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "vk_plan_get_systems": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_plan_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "vk_plan_stage_ms": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "vk_fit_variogram_samples": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                           C.c_int32, C.c_int64, C.c_uint64, C.c_void_p,
                                           C.c_void_p]),
    "vk_sample_pairs": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p,
                                  C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]),
    "vk_grid_scan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                               C.c_void_p]),
    "vk_gather_planes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64,
                                   C.c_void_p, C.c_void_p]),
    "vk_comm_unique_id": (C.c_int, [C.c_void_p]),
    "vk_comm_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "vk_comm_destroy": (C.c_int, [C.c_void_p]),
    "vk_halo_exchange": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "vk_gather_core": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_fill_generic": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_void_p, C.c_double, C.c_double,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_solve_systems": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_copy_h2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "vk_plan_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_crc32": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32, C.POINTER(C.c_uint32), C.c_void_p]),
    "vk_packbits": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vk_unpackbits": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vk_decode_samples": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]),
    "vk_normalize_stack": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vk_status_string": (C.c_char_p, [C.c_int]),
    "vk_last_error": (C.c_char_p, []),
    "vk_abi_version": (C.c_int, []),
}

_LIB = None


def load(path: os.PathLike | None = None):
    """Load (once) and return the native library; raise if it is absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeLibraryMissing(
            f"{p} is not built; run `python -m paper_2303_09523_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:
        raise NativeLibraryMissing(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.vk_abi_version() != 1:
        raise NativeLibraryMissing("ABI version mismatch")
    if path is None:
        _LIB = lib
    return lib


def last_error() -> str:
    return load().vk_last_error().decode(errors="replace")
