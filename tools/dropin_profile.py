"""Where the reference-shaped drop-in calls spend their time on one C4
sub-part (development tool).   python tools/dropin_profile.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2303_09523_b200 import VolumeGrid, fill_missing, fit_variogram
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes

cfg = CONFIGS["C4"]
planes = phantom_planes(cfg, cfg.known_z)
b, e = 0, 8
data = np.full(((e - b) * cfg.factor + 1, cfg.height, cfg.width), np.nan, dtype=np.float32)
data[::cfg.factor] = planes[b:e + 1]
mask = np.isnan(data)
kz, ky, kx = np.nonzero(~mask)
samples = (np.column_stack([kx, ky, kz]).astype(np.float64), data[kz, ky, kx].astype(np.float64))
grid = VolumeGrid(data, mask)


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms")
    return r


model = t("fit_variogram", lambda: fit_variogram(samples, "exponential"))
t("fill_missing", lambda: fill_missing(grid, model))
t("coords+values .cuda() (pageable)", lambda: (torch.from_numpy(samples[0]).cuda(), torch.from_numpy(samples[1]).cuda()))
t("grid+mask .cuda() (pageable)", lambda: (torch.from_numpy(data).cuda(), torch.from_numpy(mask.view(np.uint8)).cuda()))
d_out = torch.from_numpy(data).cuda()
t("grid .cpu() (pageable)", lambda: d_out.cpu())
pin = torch.empty(data.shape, dtype=torch.float32).pin_memory()
t("grid pinned D2H", lambda: pin.copy_(d_out))
t("np.copy of the grid", lambda: data.copy())

import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    fill_missing(grid, model)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
