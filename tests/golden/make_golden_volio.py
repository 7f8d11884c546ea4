"""Golden files of the binary volume format written by the LIVE reference
(volkrig.io.save_volume, io.py:146-167) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_volio.py

Writes tests/golden/ref_volume_{a,b,c}.vkv and reference_volio.npz (the
grids they were made from).  Tests never read /root/reference.
"""

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def grids():
    r = np.random.default_rng(146)
    a = r.normal(size=(5, 6, 7)).astype(np.float32) * 100
    ma = r.random(a.shape) < 0.4
    a[ma] = np.nan
    b = (np.arange(3 * 5 * 7, dtype=np.float32).reshape(3, 5, 7) - 50.5)   # 105 voxels: padded mask byte
    mb = np.zeros(b.shape, bool)
    c = r.normal(size=(9, 4, 3)).astype(np.float32)
    mc = np.ones(c.shape, bool)
    mc[::4] = False
    c[mc] = np.nan
    return {"a": (a, ma, (1, -2, 3)), "b": (b, mb, (0, 0, 0)), "c": (c, mc, (-7, 11, 2**20))}


def main():
    from volkrig.io import save_volume
    from volkrig.model import VolumeGrid
    blob = {}
    for k, (d, m, o) in grids().items():
        save_volume(VolumeGrid(d, m, o), os.path.join(HERE, f"ref_volume_{k}.vkv"))
        blob[f"{k}/data"], blob[f"{k}/mask"], blob[f"{k}/origin"] = d, m, np.array(o)
    np.savez(os.path.join(HERE, "reference_volio.npz"), **blob)


if __name__ == "__main__":
    main()
