"""Where the time of the reference-shaped drop-in calls goes (one C4 sub-part):
fit_variogram((coords, values)) and fill_missing(VolumeGrid(host NaN grid))
split into their host->device copies, device work and host-side steps.
Run on the GPU box: ``python tools/dropin_profile.py [--config C4]``."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2303_09523_b200 import VolumeGrid, fill_missing, fit_variogram
    from paper_2303_09523_b200 import kriging as KR
    from paper_2303_09523_b200.phantoms import CONFIGS, known_slices
    cfg = CONFIGS[args.config]
    ks = known_slices(cfg)
    q = cfg.n_known // cfg.n_subparts
    data = np.full((q * cfg.factor + 1, cfg.height, cfg.width), np.nan, dtype=np.float32)
    data[::cfg.factor] = ks[:q + 1]
    mask = np.isnan(data)
    kz, ky, kx = np.nonzero(~mask)
    coords = np.column_stack([kx, ky, kz]).astype(np.float64)
    values = data[kz, ky, kx].astype(np.float64)
    grid = VolumeGrid(data, mask)
    sync = torch.cuda.synchronize

    def t(fn):
        best = 1e9
        for _ in range(args.reps):
            sync()
            t0 = time.perf_counter()
            fn()
            sync()
            best = min(best, time.perf_counter() - t0)
        return round(1e3 * best, 3)

    fill_missing(grid, fit_variogram((coords, values)))        # warm
    res = {}
    res["fit_variogram"] = t(lambda: fit_variogram((coords, values)))
    res["fit.h2d_coords_pageable"] = t(lambda: torch.from_numpy(coords).cuda())
    res["fit.h2d_values_pageable"] = t(lambda: torch.from_numpy(values).cuda())
    res["fit.as_arrays"] = t(lambda: KR._as_coord_value_arrays((coords, values)))
    c_d = torch.from_numpy(coords).cuda()
    v_d = torch.from_numpy(values).cuda()
    lib = KR._lib.load()
    out = np.zeros(3)
    res["fit.device_call"] = t(lambda: lib.vk_fit_variogram_samples(
        c_d.data_ptr(), v_d.data_ptr(), len(values), 0, 15, 100000, 0, out.ctypes.data,
        KR._stream_handle(None)))
    model = fit_variogram((coords, values))
    res["fill_missing"] = t(lambda: fill_missing(grid, model))
    res["fill.h2d_data_pageable"] = t(lambda: torch.from_numpy(data).cuda())
    res["fill.h2d_mask_pageable"] = t(lambda: torch.from_numpy(mask.view(np.uint8)).cuda())
    res["fill.h2d_data_staged"] = t(lambda: KR._upload(data))
    res["fill.h2d_mask_staged"] = t(lambda: KR._upload(mask.view(np.uint8)))
    res["fit.h2d_coords_staged"] = t(lambda: KR._upload(coords))
    res["fill.grid_parts"] = t(lambda: KR._grid_parts(grid))
    d_d = torch.from_numpy(data).cuda()
    m_d = torch.from_numpy(mask.view(np.uint8)).cuda()
    res["fill.scan"] = t(lambda: KR._scan_grid(d_d, m_d))
    out_d = torch.empty_like(d_d)
    res["fill.d2h_pinned"] = t(lambda: torch.empty(tuple(out_d.shape), dtype=out_d.dtype,
                                                   pin_memory=True).copy_(out_d))
    res["fill.result_grid"] = t(lambda: KR._result(grid, out_d, None, False, (0, 0, 0), False))
    # the bench's loop: 4 distinct sub-parts, 2 reps, per-call times
    grids = []
    for b in range(0, 4 * q, q):
        d = np.full((q * cfg.factor + 1, cfg.height, cfg.width), np.nan, dtype=np.float32)
        d[::cfg.factor] = ks[b:b + q + 1]
        grids.append(VolumeGrid(d, np.isnan(d)))
    seq = []
    for _ in range(2):
        for g in grids:
            sync()
            t0 = time.perf_counter()
            o = fill_missing(g, model)
            sync()
            seq.append(round(1e3 * (time.perf_counter() - t0), 2))
    res["fill_missing_bench_loop"] = seq
    res["bytes"] = {"coords": coords.nbytes, "values": values.nbytes, "data": data.nbytes,
                    "mask": mask.nbytes}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
