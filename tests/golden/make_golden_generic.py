"""Generate golden vectors for the generic per-voxel path (non-plane masks)
from the LIVE reference (volkrig.kriging.fill_missing, kriging.py:458-496,
408-431), run in the build container where /root/reference is mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_generic.py

Writes tests/golden/reference_generic.npz (+ .json with the environment).
The GPU box never reads /root/reference; tests read only the committed files.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    r = np.random.default_rng(2303)

    def field(T, H, W, lo=20.0, span=200.0):
        b = r.normal(size=(T, H, W)).cumsum(0).cumsum(1).cumsum(2)
        b = (b - b.min()) / (b.max() - b.min()) * span + lo
        return b.astype(np.float32)

    out = []
    # 1. random dropout 30 %, linear drift, variance
    d = field(9, 10, 12)
    m = r.random(d.shape) < 0.3
    out.append(("dropout30_linear", d, m, ("exponential", 0.5, 400.0, 6.0), "linear"))
    # 2. random dropout 70 %, ordinary kriging
    d = field(8, 11, 9)
    m = r.random(d.shape) < 0.7
    out.append(("dropout70_constant", d, m, ("exponential", 0.0, 300.0, 5.0), "constant"))
    # 3. whole missing planes plus a missing rectangle inside a known plane
    d = field(13, 12, 14)
    m = np.zeros(d.shape, bool)
    m[1::2] = True
    m[4, 3:9, 2:7] = True
    out.append(("planes_plus_hole", d, m, ("exponential", 1.0, 500.0, 8.0), "linear"))
    # 4. sparse known lattice: windows widen to (8, 16) / (16, 16)
    d = field(18, 20, 19)
    m = np.ones(d.shape, bool)
    m[::5, ::6, ::6] = False
    out.append(("sparse_lattice", d, m, ("exponential", 0.2, 250.0, 10.0), "linear"))
    # 5. gaussian and spherical kinds on a column dropout
    d = field(10, 9, 11)
    m = np.zeros(d.shape, bool)
    m[:, :, 4] = True
    m[3:7, 5, :] = True
    out.append(("columns_gaussian", d, m, ("gaussian", 0.3, 350.0, 7.0), "linear"))
    out.append(("columns_spherical", d, m, ("spherical", 0.3, 350.0, 7.0), "constant"))
    # 6. a single known z-column plus noise dropout in a thin volume
    d = field(6, 5, 16)
    m = r.random(d.shape) < 0.5
    m[:, 2, :] = True
    out.append(("thin_rows", d, m, ("exponential", 0.0, 100.0, 4.0), "linear"))
    return out


def main():
    from volkrig import kriging as K
    from volkrig.errors import NoKnownNeighbors
    from volkrig.model import VolumeGrid
    blob, meta = {}, {"cases": []}
    for name, d, m, (kind, nug, sill, rng_), drift in cases():
        data = d.copy()
        data[m] = np.nan
        g, v = K.fill_missing(VolumeGrid(data, m), K.VariogramModel(kind, nug, sill, rng_), drift,
                              return_variance=True)
        blob[f"{name}/data"] = data
        blob[f"{name}/mask"] = m
        blob[f"{name}/out"] = g.data
        blob[f"{name}/var"] = v
        meta["cases"].append({"name": name, "model": [kind, nug, sill, rng_], "drift": drift,
                              "shape": list(d.shape), "n_missing": int(m.sum())})
    # interpolate_voxel (kriging.py:384-405) on the first case's grid: a few
    # targets x windows, own RNG so the cases above do not move
    name0, d0, m0, (kind0, nug0, sill0, rng0), drift0 = cases()[0]
    data0 = d0.copy()
    data0[m0] = np.nan
    g0 = VolumeGrid(data0, m0)
    rv = np.random.default_rng(384)
    vox = []
    miss = np.argwhere(m0)
    for t in rv.choice(len(miss), 12, replace=False):
        z, y, x = (int(v) for v in miss[t])
        for inplane, z_extent in ((4, 4), (4, 8), (8, 16)):
            try:
                val = K.interpolate_voxel(g0, (x, y, z), K.VariogramModel(kind0, nug0, sill0, rng0), drift0,
                                          inplane, z_extent)
            except NoKnownNeighbors:
                val = None
            vox.append({"target": [x, y, z], "inplane": inplane, "z_extent": z_extent, "value": val})
    known = np.argwhere(~m0)[0]
    vox.append({"target": [int(known[2]), int(known[1]), int(known[0])], "inplane": 4, "z_extent": 4,
                "value": float(data0[tuple(known)])})
    meta["interpolate_voxel"] = {"case": name0, "voxels": vox}
    # NoKnownNeighbors: nothing known within the widest window of x = 39
    data = np.full((1, 1, 40), np.nan, np.float32)
    data[0, 0, 0] = 5.0
    mask = np.isnan(data)
    try:
        K.fill_missing(VolumeGrid(data, mask), K.VariogramModel("exponential", 0.0, 1.0, 3.0))
        meta["no_neighbors"] = None
    except NoKnownNeighbors as exc:
        meta["no_neighbors"] = {"shape": [1, 1, 40], "known_x": 0, "message": str(exc)}
    import scipy
    meta["env"] = {"numpy": np.__version__, "scipy": scipy.__version__, "python": sys.version.split()[0]}
    np.savez_compressed(os.path.join(HERE, "reference_generic.npz"), **blob)
    with open(os.path.join(HERE, "reference_generic.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
