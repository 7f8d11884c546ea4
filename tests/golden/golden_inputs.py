"""Seeded input generators shared by make_golden.py (which runs the live
reference) and the tests (which regenerate the same inputs).  No reference
imports here: this module travels to the GPU box."""

import numpy as np


def smooth_grid(seed, T, H, W, known_z, quant=True):
    """Seeded smooth random volume with NaN planes except known_z."""
    r = np.random.default_rng(seed)
    base = r.normal(size=(T, H, W)).cumsum(1).cumsum(2)
    base = (base - base.min()) / (base.max() - base.min()) * 200 + 20
    if quant:
        base = np.rint(base)
    data = base.astype(np.float32)
    mask = np.ones(data.shape, bool)
    mask[list(known_z)] = False
    data[mask] = np.nan
    return data, mask
