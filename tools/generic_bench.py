"""Throughput of the device generic per-voxel path (non-plane masks) on a
random-dropout volume; prints JSON (distinct systems, time, voxels/s)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_09523_b200 import _lib  # noqa: E402

lib = _lib.load()
for (T, H, W, frac, planes) in [(33, 128, 128, 0.1, False), (33, 256, 256, 0.02, False),
                                (65, 256, 256, 0.0, True)]:
    r = np.random.default_rng(0)
    base = r.normal(size=(T, H, W)).cumsum(1).cumsum(2).astype(np.float32)
    mask = r.random(base.shape) < frac
    if planes:                                   # plane layout with a hole in each known plane
        mask[np.arange(T) % 4 != 0] = True
        mask[::4, 100:110, 100:110] = True
    data = np.where(mask, np.nan, base).astype(np.float32)
    d = torch.from_numpy(data).cuda()
    m = torch.from_numpy(mask.view(np.uint8)).cuda()
    out = torch.empty_like(d)
    model = np.array([0.5, 50.0, 8.0])
    info = np.zeros(3, np.int64)
    lo, hi = float(np.nanmin(data)), float(np.nanmax(data))
    args = (d.data_ptr(), m.data_ptr(), T, H, W, 0, 0, model.ctypes.data, lo, hi, out.data_ptr(), None,
            info.ctypes.data, None)
    assert lib.vk_fill_generic(*args) == 0, lib.vk_last_error()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = lib.vk_fill_generic(*args)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"shape": [T, H, W], "dropout": frac, "planes_with_holes": planes, "status": st,
                      "missing": int(info[2]), "distinct_systems": int(info[1]), "seconds": dt,
                      "voxels_per_s": info[2] / dt}), flush=True)
