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


def _reference_classes():
    try:
        import sys
        sys.path.insert(0, "/root/reference/pkg/src")
        from volkrig.kriging import VariogramModel as RM
        from volkrig.model import VolumeGrid as RG
        return [(RG, RM)]
    except Exception:
        return []


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
