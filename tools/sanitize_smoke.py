"""Small end-to-end exercise of every device path, sized for
compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_09523_b200 import (BlockKriging, VariogramModel, VolumeGrid, ZPartKriging,  # noqa: E402
                                   fill_missing, fit_variogram, interpolate_voxel, load_volume,
                                   save_volume, solve_systems)
from paper_2303_09523_b200.phantoms import known_slices, small_config  # noqa: E402

cfg = small_config("head", 40, 136, 9, 8, n_subparts=3, seed=3)     # G = 7, odd height, 2 x-tiles
ks = torch.from_numpy(known_slices(cfg)).cuda()
for accum in ("fp64", "fp32", "fixed"):
    for overlap in (True, False):
        zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, accum=accum,
                          overlap=overlap)
        zk.run(ks, return_variance=True)
        zk.finish()
cfg4 = small_config("brain", 33, 64, 9, 4, n_subparts=2, seed=4)     # G = 3 (three CTAs per SM)
zk = ZPartKriging(cfg4.n_known, cfg4.height, cfg4.width, cfg4.factor, cfg4.n_subparts, accum="fp32")
zk.run(torch.from_numpy(known_slices(cfg4)).cuda())
zk.finish()
r = np.random.default_rng(0)
data = r.normal(size=(7, 12, 13)).cumsum(2).astype(np.float32)
mask = r.random(data.shape) < 0.3
data[mask] = np.nan
m = VariogramModel("exponential", 0.1, 2.0, 5.0)
fill_missing(VolumeGrid(data, mask), m, return_variance=True)                  # generic path
interpolate_voxel(VolumeGrid(data, mask), tuple(int(v) for v in np.argwhere(mask)[0][::-1]), m)
solve_systems([np.array([[1, 0, 0], [0, 1, 0], [-1, 0, 1], [0, 0, -1]])], m)
fit_variogram((r.random((500, 3)) * 10, r.random(500)))
bk = BlockKriging(9, 48, 64, 2, k=2, halo_width=4)
bk.run(torch.from_numpy(known_slices(small_config("spine", 48, 64, 9, 2, seed=5))).cuda())
bk.finish()
with tempfile.TemporaryDirectory() as d:
    save_volume(VolumeGrid(data, mask, (1, 2, 3)), os.path.join(d, "v.vkv"))
    load_volume(os.path.join(d, "v.vkv"))
torch.cuda.synchronize()
print("sanitize_smoke ok")
