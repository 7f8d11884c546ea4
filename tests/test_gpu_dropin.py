"""GPU: the drop-in entry points accept the reference's own boundary types.

INTEGRATION.md's switch hands ``fill_missing`` / ``interpolate_voxel`` the
objects a reference caller already has: ``volkrig.model.VolumeGrid``
(model.py:71-129: ``.data``, ``.missing_mask``, ``.origin_offset``, ``.copy``)
and ``volkrig.kriging.VariogramModel`` (kriging.py:44-57: ``.kind``,
``.nugget``, ``.sill``, ``.range_len``).  The reference cannot travel to the
GPU box, so RefGrid / RefModel below restate exactly that attribute surface
(no torch, no ``as_array``, no ``on_device``); when the live reference is
importable (build container with a GPU) its classes are used as well.
Also: a plane mask whose z window reaches more than NPMAX = 8 known planes
(the streaming plan refuses it) goes to the device per-voxel path and still
matches the oracle.
"""

import os
import sys
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import kriging_oracle as O

pytestmark = pytest.mark.gpu


@dataclass
class RefGrid:                     # model.py:71-129 attribute surface
    data: np.ndarray
    missing_mask: np.ndarray = None
    origin_offset: tuple = (0, 0, 0)

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float32)
        if self.missing_mask is None:
            self.missing_mask = np.isnan(self.data)
        self.missing_mask = np.ascontiguousarray(self.missing_mask, dtype=bool)

    def copy(self):
        return RefGrid(self.data.copy(), self.missing_mask.copy(), self.origin_offset)


@dataclass
class RefModel:                    # kriging.py:44-57 attribute surface
    kind: str
    nugget: float
    sill: float
    range_len: float


def _grid(seed=3, T=13, H=24, W=32, f=4):
    rng = np.random.default_rng(seed)
    data = rng.normal(100.0, 20.0, (T, H, W)).astype(np.float32)
    data = np.rint(data)
    mask = np.ones((T, H, W), bool)
    mask[::f] = False
    data[mask] = np.nan
    return data, mask


REF_INSTALL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _volkrig():
    """The unmodified reference: the git-ignored baseline/_ref install that
    travels with the snapshot (tools/vendor_ref.py), else the mounted source
    tree (build container); None when neither is there."""
    for path in (REF_INSTALL, "/root/reference/pkg/src"):
        if os.path.isfile(os.path.join(path, "volkrig", "kriging.py")):
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import volkrig.kriging as K
                import volkrig.model as M
                return K, M
            except Exception:
                return None
    return None


def _reference_classes():
    vk = _volkrig()
    return [(vk[1].VolumeGrid, vk[0].VariogramModel)] if vk else []


@pytest.mark.parametrize("classes", [(RefGrid, RefModel)] + _reference_classes(),
                         ids=lambda c: c[0].__module__)
def test_fill_missing_accepts_reference_types(cuda, classes):
    from paper_2303_09523_b200 import VariogramModel, VolumeGrid, fill_missing
    G, M = classes
    data, mask = _grid()
    ref_grid = G(data.copy(), mask.copy(), (5, 6, 7))
    ref_model = M("exponential", 1.0, 400.0, 15.0)
    got, var = fill_missing(ref_grid, ref_model, "linear", True)
    assert type(got) is G
    assert got.origin_offset == (5, 6, 7)
    assert not got.missing_mask.any()
    ours, var2 = fill_missing(VolumeGrid(data, mask, (5, 6, 7)), VariogramModel("exponential", 1.0, 400.0, 15.0),
                              "linear", True)
    assert np.array_equal(got.data, ours.data) and np.array_equal(var, var2)
    exp, _ = O.fill_missing(data, mask, O.Model("exponential", 1.0, 400.0, 15.0))
    rng = float(np.nanmax(data) - np.nanmin(data))
    assert np.abs(got.data.astype(np.float64) - exp).max() <= 1e-6 * rng
    # dense grid: returned as the caller's own copy
    dense = G(np.ones((3, 4, 5), np.float32), np.zeros((3, 4, 5), bool))
    d2 = fill_missing(dense, ref_model)
    assert type(d2) is G and d2 is not dense and np.array_equal(d2.data, dense.data)


def test_interpolate_voxel_and_fit_accept_reference_types(cuda):
    from paper_2303_09523_b200 import fit_variogram, interpolate_voxel
    data, mask = _grid(seed=5)
    g = RefGrid(data, mask)
    m = RefModel("exponential", 0.5, 300.0, 12.0)
    v = interpolate_voxel(g, (10, 9, 2), m, "linear")
    assert np.isfinite(v)
    kz, ky, kx = np.nonzero(~mask)
    samples = (np.column_stack([kx, ky, kz]).astype(np.float64), data[kz, ky, kx].astype(np.float64))
    got = fit_variogram(samples)
    exp = O.fit_variogram(samples)
    assert abs(got.nugget - exp.nugget) <= 1e-7 * exp.sill
    assert abs(got.sill - exp.sill) <= 1e-6 * exp.sill
    assert abs(got.range_len - exp.range_len) <= 1e-4 * exp.range_len


def test_plane_mask_beyond_npmax_takes_the_per_voxel_path(cuda):
    """Known planes everywhere but z = 10..16: the missing plane z = 13 is
    bracketed only at z extent 16, whose window holds 9 known planes (> NPMAX),
    so the streaming plan is refused; the per-voxel path selects the same
    windows (kriging.py:444-455 vs 408-431) and matches the oracle's
    plane-structured fill."""
    from paper_2303_09523_b200 import fill_missing
    rng = np.random.default_rng(11)
    T, H, W = 26, 12, 16
    data = np.rint(rng.normal(50.0, 10.0, (T, H, W))).astype(np.float32)
    mask = np.zeros((T, H, W), bool)
    mask[10:17] = True
    data[mask] = np.nan
    model = RefModel("exponential", 0.5, 150.0, 8.0)
    got = fill_missing(RefGrid(data, mask), model)
    exp, _ = O.fill_missing(data, mask, O.Model("exponential", 0.5, 150.0, 8.0))
    rng_ = float(np.nanmax(data) - np.nanmin(data))
    assert np.abs(got.data.astype(np.float64) - exp).max() <= 1e-6 * rng_


def test_integration_switch_against_the_live_reference(cuda):
    """INTEGRATION.md section 1 verbatim on the unmodified reference: its own
    VolumeGrid and its own fit_variogram output go into our fill_missing; the
    result matches the reference's fill_missing at the fp64 gate, and our
    fit_variogram reproduces its fit (kriging.py:264-328, 458-496)."""
    vk = _volkrig()
    if vk is None:
        pytest.skip("reference not installed (python tools/vendor_ref.py)")
    K, M = vk
    from paper_2303_09523_b200 import fill_missing, fit_variogram
    for seed, drift in ((21, "linear"), (22, "constant")):
        data, mask = _grid(seed=seed)
        grid = M.VolumeGrid(data.copy(), mask.copy())
        kz, ky, kx = np.nonzero(~mask)
        samples = (np.column_stack([kx, ky, kz]).astype(np.float64), data[kz, ky, kx].astype(np.float64))
        ref_model = K.fit_variogram(samples)
        expect = K.fill_missing(grid, ref_model, drift=drift)
        got = fill_missing(grid, ref_model, drift)
        assert type(got) is M.VolumeGrid
        rng = float(np.nanmax(data) - np.nanmin(data))
        err = np.abs(got.data.astype(np.float64) - expect.data.astype(np.float64)).max()
        assert err <= 1e-6 * rng, (seed, drift, err / rng)
        known = ~mask
        assert np.array_equal(got.data[known], expect.data[known])
        ours = fit_variogram(samples)
        assert abs(ours.nugget - ref_model.nugget) <= 1e-7 * ref_model.sill
        assert abs(ours.sill - ref_model.sill) <= 1e-6 * ref_model.sill
        assert abs(ours.range_len - ref_model.range_len) <= 1e-4 * ref_model.range_len


@pytest.mark.parametrize("nbytes,offset", [(0, 0), (1, 3), (1 << 20, 0), ((1 << 20) - 1, 5),
                                           ((4 << 20) + 3, 1), ((13 << 20) + 5, 7)])
def test_staged_upload_is_byte_exact(cuda, nbytes, offset):
    """vk_copy_h2d (the drop-in's host -> device path) at sizes around its
    pageable / staged switch and its 4 MB chunks, from unaligned sources."""
    import torch
    from paper_2303_09523_b200 import _lib
    from paper_2303_09523_b200.kriging import _stream_handle
    rng = np.random.default_rng(nbytes)
    buf = rng.integers(0, 256, nbytes + offset + 16, dtype=np.uint8)
    src = buf[offset:offset + nbytes]
    expect = src.copy()
    dst = torch.full((nbytes + 16,), 0xAB, dtype=torch.uint8, device="cuda")
    assert _lib.load().vk_copy_h2d(dst.data_ptr(), src.ctypes.data, nbytes, _stream_handle(None)) == 0
    buf[offset:offset + nbytes] = 0                 # the source may be reused once the call returns
    got = dst.cpu().numpy()
    assert np.array_equal(got[:nbytes], expect)
    assert (got[nbytes:] == 0xAB).all()
