"""GPU parity of the generic per-voxel path (masks that are not whole known /
missing planes; kriging.py:408-431) against golden vectors produced by the
LIVE reference (tests/golden/make_golden_generic.py) and against the oracle's
restatement (oracle.fill_generic): max-abs <= 1e-6 of the known range, known
voxels bit-exact, variance rtol 1e-9, NoKnownNeighbors on the same voxel."""

import json
import os

import numpy as np
import pytest

from oracle import kriging_oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
TOL64 = 1e-6


def _golden():
    d = np.load(os.path.join(HERE, "golden", "reference_generic.npz"))
    with open(os.path.join(HERE, "golden", "reference_generic.json")) as f:
        return d, json.load(f)


def _model(c):
    from paper_2303_09523_b200 import VariogramModel
    kind, nug, sill, rng = c["model"]
    return VariogramModel(kind, nug, sill, rng)


@pytest.mark.parametrize("name", [c["name"] for c in _golden()[1]["cases"]])
def test_generic_vs_reference_goldens(cuda, name):
    from paper_2303_09523_b200 import VolumeGrid, fill_missing
    d, meta = _golden()
    c = next(c for c in meta["cases"] if c["name"] == name)
    data, mask = d[f"{name}/data"], d[f"{name}/mask"]
    got, var = fill_missing(VolumeGrid(data, mask), _model(c), c["drift"], return_variance=True)
    ref, rvar = d[f"{name}/out"], d[f"{name}/var"]
    rng = float(np.nanmax(data) - np.nanmin(data))
    assert np.array_equal(got.data[~mask], data[~mask])
    assert not got.missing_mask.any()
    err = np.abs(got.data.astype(np.float64) - ref).max() / rng
    assert err <= TOL64, err
    assert np.abs(np.rint(got.data) - np.rint(ref)).max() <= 1
    assert np.allclose(var, rvar, rtol=1e-9, atol=1e-9 * c["model"][2])
    assert np.all(var[~mask] == 0)


def test_generic_no_known_neighbors(cuda):
    from paper_2303_09523_b200 import VariogramModel, VolumeGrid, fill_missing
    from paper_2303_09523_b200.errors import NoKnownNeighbors
    _, meta = _golden()
    nn = meta["no_neighbors"]
    data = np.full(nn["shape"], np.nan, np.float32)
    data[0, 0, nn["known_x"]] = 5.0
    with pytest.raises(NoKnownNeighbors, match=r"\(8, 0, 0\)"):
        fill_missing(VolumeGrid(data, np.isnan(data)), VariogramModel("exponential", 0.0, 1.0, 3.0))


@pytest.mark.parametrize("frac,drift", [(0.2, "linear"), (0.6, "constant"), (0.9, "linear")])
def test_generic_random_masks_vs_oracle(cuda, frac, drift):
    """Larger random masks on a device-resident grid (torch in, torch out)."""
    torch = cuda
    from paper_2303_09523_b200 import VariogramModel, VolumeGrid, fill_missing
    r = np.random.default_rng(int(frac * 100))
    T, H, W = 14, 24, 22
    base = r.normal(size=(T, H, W)).cumsum(1).cumsum(2)
    base = ((base - base.min()) / (base.max() - base.min()) * 300 + 10).astype(np.float32)
    mask = r.random(base.shape) < frac
    data = base.copy()
    data[mask] = np.nan
    m = VariogramModel("exponential", 0.5, 250.0, 9.0)
    g = VolumeGrid(torch.from_numpy(data).cuda(), torch.from_numpy(mask).cuda())
    got, var = fill_missing(g, m, drift, return_variance=True)
    assert got.data.is_cuda and var.is_cuda
    ref, rvar = O.fill_missing(data, mask, O.Model("exponential", 0.5, 250.0, 9.0), drift, True)
    rng = float(base[~mask].max() - base[~mask].min())
    err = np.abs(got.data.cpu().numpy().astype(np.float64) - ref).max() / rng
    assert err <= TOL64, err
    assert np.allclose(var.cpu().numpy(), rvar, rtol=1e-9, atol=1e-9 * 250.0)


def test_generic_planes_with_holes_vs_oracle(cuda):
    """Mostly plane-structured data with a few partial planes: the whole grid
    takes the generic path (kriging.py:485-490), as in the reference."""
    from paper_2303_09523_b200 import VariogramModel, VolumeGrid, fill_missing
    r = np.random.default_rng(5)
    T, H, W = 17, 20, 18
    base = r.normal(size=(T, H, W)).cumsum(0).cumsum(2)
    base = ((base - base.min()) / (base.max() - base.min()) * 4095).astype(np.float32)
    mask = np.zeros(base.shape, bool)
    mask[np.arange(T) % 4 != 0] = True
    mask[8, 5:12, 3:15] = True                      # hole in a known plane
    mask[12, :, 0] = True
    data = base.copy()
    data[mask] = np.nan
    got = fill_missing(VolumeGrid(data, mask), VariogramModel("exponential", 1.0, 9e5, 12.0))
    ref, _ = O.fill_missing(data, mask, O.Model("exponential", 1.0, 9e5, 12.0))
    rng = float(base[~mask].max() - base[~mask].min())
    assert np.abs(got.data.astype(np.float64) - ref).max() <= TOL64 * rng


def test_solve_systems_vs_reference_solve_ked(cuda):
    """vk_solve_systems on the 672 stencil systems the live reference solved
    with build_system + solve_ked (tests/golden/make_golden.py), batched by
    model and drift."""
    from paper_2303_09523_b200 import VariogramModel, solve_systems
    gold = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
    with open(os.path.join(HERE, "golden", "reference_golden.json")) as f:
        meta = json.load(f)
    groups = {}
    for s in meta["systems"]:
        groups.setdefault((tuple(s["model"]), s["drift"]), []).append(s)
    worst_w = worst_v = 0.0
    for (model, drift), sys_ in groups.items():
        kind, nug, sill, rng = model
        ws, vs = solve_systems([gold[f"sys_{s['id']}_rel"] for s in sys_],
                               VariogramModel(kind, nug, sill, rng), drift)
        for s, w, v in zip(sys_, ws, vs):
            ref = gold[f"sys_{s['id']}_w"]
            worst_w = max(worst_w, float(np.abs(w - ref).max() / max(1.0, np.abs(ref).max())))
            worst_v = max(worst_v, abs(v - s["variance"]) / max(abs(s["variance"]), 1e-12 * sill))
    assert worst_w <= 1e-7, worst_w
    assert worst_v <= 1e-7, worst_v


def test_interpolate_voxel_vs_reference(cuda):
    from paper_2303_09523_b200 import VolumeGrid, interpolate_voxel
    d, meta = _golden()
    iv = meta["interpolate_voxel"]
    c = next(c for c in meta["cases"] if c["name"] == iv["case"])
    data, mask = d[f"{iv['case']}/data"], d[f"{iv['case']}/mask"]
    grid = VolumeGrid(data, mask)
    rng = float(np.nanmax(data) - np.nanmin(data))
    for v in iv["voxels"]:
        got = interpolate_voxel(grid, v["target"], _model(c), c["drift"], v["inplane"], v["z_extent"])
        assert abs(got - v["value"]) <= 1e-9 * rng, (v, got)
