"""CPU oracle for slice-stack decode + normalisation -- TEST INFRASTRUCTURE ONLY.

Restates in numpy what the reference's ``load_stack`` does to the decoded
samples (``_decode_slice``, io.py:108-125; ``normalize_stack``,
model.py:189-202) so the device path (``vk_decode_samples`` /
``vk_normalize_stack``) can be checked bit for bit on the GPU box.  Image
decoding itself is Pillow on the host in both the reference and the product,
so the oracle starts from Pillow's sample arrays.  Pinned against the live
reference's outputs (``tests/golden/make_golden_stack.py`` ->
``tests/golden/reference_stack.npz``, ``tests/test_stack_io.py``).  Only
``tests/`` may import this module.
"""

from __future__ import annotations

import numpy as np
from PIL import Image


def slice_samples(img: "Image.Image"):
    """Pillow image -> (integer sample array, scale) as io.py:112-121 reads it:
    "I;16" -> u16 / 65535; "L"/"P"/"1" -> convert("L") / 255; "I" -> i32 / 65535;
    anything else -> convert("L") / 255."""
    if img.mode == "I;16":
        return np.asarray(img, dtype=np.uint16), 65535.0
    if img.mode == "I":
        return np.asarray(img, dtype=np.int32), 65535.0
    return np.asarray(img.convert("L"), dtype=np.uint8), 255.0


def decode(samples: np.ndarray, scale: float) -> np.ndarray:
    """f32(sample) / scale in float32 (io.py:113-119: the python float divisor
    is weakly typed under NumPy 2, so the division is an f32 division)."""
    return samples.astype(np.float32) / np.float32(scale)


def normalize(data: np.ndarray) -> np.ndarray:
    """model.py:194-201: (data - lo) / (hi - lo) in float32, lo/hi the global
    extremes as python floats; all zeros for a constant stack."""
    data = np.asarray(data, dtype=np.float32)
    lo = float(data.min())
    hi = float(data.max())
    if hi > lo:
        return ((data - np.float32(lo)) / np.float32(hi - lo)).astype(np.float32)
    return np.zeros_like(data)


def load_samples(paths):
    """Decode every slice of a manifest on the host, reference order."""
    out = []
    for p in paths:
        with Image.open(p) as img:
            img.load()
            out.append(decode(*slice_samples(img)))
    return normalize(np.stack(out))
