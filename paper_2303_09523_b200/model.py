"""Boundary data types of the kriging path, mirroring the reference's
``volkrig.model`` (model.py:23-129, 205-217).

``VolumeGrid`` holds float32 ``[z, y, x]`` data with an authoritative missing
mask and the NaN sentinel; it accepts numpy arrays (the reference's type) and
also CUDA ``torch`` tensors, which lets device-resident volumes enter the
kriging path without a host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch, EmptyStack, NonPositiveSpacing

AXIS_LABELS = ("axial", "sagittal", "coronal")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def missing_planes_per_gap(slice_gap_mm: float, pixel_spacing_mm: float) -> int:
    """g = max(0, floor(gap/spacing + 0.5) - 1) -- model.py:205-217."""
    if slice_gap_mm <= 0 or pixel_spacing_mm <= 0:
        raise NonPositiveSpacing("gap and spacing must be > 0")
    return max(0, int(np.floor(slice_gap_mm / pixel_spacing_mm + 0.5)) - 1)


def check_stack_meta(shape, pixel_spacing, slice_gap_mm, axis_label) -> None:
    """The shape/spacing/axis checks of SliceStack.__post_init__ (model.py:37-44),
    in order; callable before any sample is on the device."""
    if len(shape) != 3 or shape[0] < 2:
        raise EmptyStack("a stack needs at least 2 slices of equal size")
    if slice_gap_mm <= 0 or min(pixel_spacing) <= 0:
        raise NonPositiveSpacing("spacing and gap must be > 0")
    if axis_label not in AXIS_LABELS:
        raise ValueError(f"axis_label must be one of {AXIS_LABELS}")


@dataclass
class SliceStack:
    """Registered 2D slices along one axis -- model.py:23-68.  ``slices`` is a
    float32 ``[n, h, w]`` numpy array or CUDA tensor (``load_stack`` returns
    the device form)."""

    slices: np.ndarray
    pixel_spacing: tuple[float, float]
    slice_gap_mm: float
    axis_label: str = "axial"

    def __post_init__(self):
        if _is_torch(self.slices):
            import torch
            self.slices = self.slices.to(torch.float32).contiguous()
        else:
            self.slices = np.ascontiguousarray(self.slices, dtype=np.float32)
        check_stack_meta(tuple(self.slices.shape), self.pixel_spacing, self.slice_gap_mm, self.axis_label)
        if _is_torch(self.slices):
            import torch
            finite = bool(torch.isfinite(self.slices).all())
        else:
            finite = bool(np.isfinite(self.slices).all())
        if not finite:
            raise ValueError("slice values must be finite")

    @property
    def on_device(self) -> bool:
        return _is_torch(self.slices)

    @property
    def n(self) -> int:
        return self.slices.shape[0]

    @property
    def height(self) -> int:
        return self.slices.shape[1]

    @property
    def width(self) -> int:
        return self.slices.shape[2]

    @property
    def missing_per_gap(self) -> int:
        return missing_planes_per_gap(self.slice_gap_mm, self.pixel_spacing[0])

    @property
    def factor(self) -> int:
        """Upsampling factor f = g + 1 (known slice i sits at z = i*f)."""
        return self.missing_per_gap + 1

    def output_depth(self) -> int:
        return self.n + (self.n - 1) * self.missing_per_gap


class VolumeGrid:
    """Dense grid with an explicit missing mask -- model.py:71-129."""

    def __init__(self, data, missing_mask=None, origin_offset=(0, 0, 0)):
        if _is_torch(data):
            import torch
            data = data.to(torch.float32).contiguous()
            if data.dim() != 3:
                raise ValueError("volume data must be 3D")
            if missing_mask is None:
                missing_mask = torch.isnan(data)
            missing_mask = missing_mask.to(torch.bool).contiguous()
            if tuple(missing_mask.shape) != tuple(data.shape):
                raise DimensionMismatch("mask shape must match data shape")
        else:
            data = np.ascontiguousarray(data, dtype=np.float32)
            if data.ndim != 3:
                raise ValueError("volume data must be 3D")
            if missing_mask is None:
                missing_mask = np.isnan(data)
            missing_mask = np.ascontiguousarray(missing_mask, dtype=bool)
            if missing_mask.shape != data.shape:
                raise DimensionMismatch("mask shape must match data shape")
        self.data = data
        self.missing_mask = missing_mask
        self.origin_offset = tuple(origin_offset)

    @property
    def on_device(self) -> bool:
        return _is_torch(self.data)

    @property
    def dims(self) -> tuple[int, int, int]:
        dz, dy, dx = self.data.shape
        return (dx, dy, dz)

    @property
    def n_voxels(self) -> int:
        dz, dy, dx = self.data.shape
        return dz * dy * dx

    def linear_index(self, x: int, y: int, z: int) -> int:
        dx, dy, _ = self.dims
        return x + dx * (y + dy * z)

    def is_dense(self) -> bool:
        return not bool(self.missing_mask.any())

    def validate(self):
        """NaN sentinel <-> mask, known voxels finite (model.py:111-117)."""
        if self.on_device:
            import torch
            nan = torch.isnan(self.data)
            if not torch.equal(nan, self.missing_mask):
                raise ValueError("missing_mask out of sync with NaN sentinel")
            if not bool(torch.isfinite(self.data[~self.missing_mask]).all()):
                raise ValueError("known voxels must be finite")
            return
        if not np.array_equal(np.isnan(self.data), self.missing_mask):
            raise ValueError("missing_mask out of sync with NaN sentinel")
        if not np.isfinite(self.data[~self.missing_mask]).all():
            raise ValueError("known voxels must be finite")

    def copy(self) -> "VolumeGrid":
        return VolumeGrid(self.data.clone() if self.on_device else self.data.copy(),
                          self.missing_mask.clone() if self.on_device
                          else self.missing_mask.copy(), self.origin_offset)

    @classmethod
    def empty(cls, dims, origin_offset=(0, 0, 0)) -> "VolumeGrid":
        dx, dy, dz = dims
        data = np.full((dz, dy, dx), np.nan, dtype=np.float32)
        return cls(data, np.ones((dz, dy, dx), dtype=bool), origin_offset)

    def __repr__(self):
        return (f"VolumeGrid(shape={tuple(self.data.shape)}, "
                f"device={'cuda' if self.on_device else 'host'}, "
                f"origin_offset={self.origin_offset})")
