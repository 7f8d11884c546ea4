"""GPU block pipeline (partition -> per-block fit + fill -> merge,
SPEC.md:381-445) against the oracle's composition: with the oracle's
per-block models at the fp64 gate, and end to end (device fits) at the fit
fuzz bound; known planes bit-exact; merge ownership."""

import numpy as np
import pytest

from oracle import kriging_oracle as O

pytestmark = pytest.mark.gpu

TOL64 = 1e-6
FIT_FUZZ = 1e-6     # device fits reproduce the reference's (test_gpu_fit_parity.py)


def _stack(seed, K, H, W):
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    return known_slices(small_config("head", H, W, K, 2, n_subparts=1, seed=seed))


@pytest.mark.parametrize("halo,tiles,f", [(4, (2, 2), 4), (2, (2, 2), 2), (4, (1, 2), 8), (4, (2, 3), 4)])
def test_blocks_vs_oracle_given_models(cuda, halo, tiles, f):
    torch = cuda
    from paper_2303_09523_b200 import VariogramModel
    from paper_2303_09523_b200.blocks import BlockKriging
    K, H, W = 9, 48, 72
    ks = _stack(halo + f, K, H, W)
    ref, models = O.reconstruct_blocks(ks, f, k=2, halo_width=halo, tiles=tiles)
    bk = BlockKriging(K, H, W, f, k=2, halo_width=halo, tiles=tiles, fit=False)
    out, _ = bk.run(torch.from_numpy(ks).cuda(),
                    models=[VariogramModel("exponential", m.nugget, m.sill, m.range_len) for m in models])
    bk.finish()
    got = out.cpu().numpy()
    assert np.array_equal(got[::f], ks)
    rng = float(ks.max() - ks.min())
    assert np.abs(got.astype(np.float64) - ref).max() <= TOL64 * rng


def test_blocks_end_to_end_with_device_fits(cuda):
    torch = cuda
    from paper_2303_09523_b200.blocks import BlockKriging
    K, H, W, f = 9, 64, 64, 4
    ks = _stack(3, K, H, W)
    ref, rmodels = O.reconstruct_blocks(ks, f, k=2, halo_width=4)
    bk = BlockKriging(K, H, W, f, k=2, halo_width=4)
    out, _ = bk.run(torch.from_numpy(ks).cuda())
    models, ranges = bk.finish()
    assert len(models) == 8 and len(ranges) == 8
    for m, r in zip(models, rmodels):
        assert abs(m.sill - r.sill) <= 1e-4 * r.sill
    got = out.cpu().numpy()
    rng = float(ks.max() - ks.min())
    assert np.abs(got.astype(np.float64) - ref).max() <= FIT_FUZZ * rng
    assert np.abs(np.rint(got) - np.rint(ref)).max() <= 1


def test_blocks_constant_and_ownership(cuda):
    """Blocks carrying their own id (constant per block) merge to the tiling
    map; a constant volume stays constant."""
    torch = cuda
    from paper_2303_09523_b200 import VariogramModel
    from paper_2303_09523_b200.blocks import BlockKriging
    K, H, W, f = 5, 32, 48, 2
    ks = np.full((K, H, W), 7.0, np.float32)
    bk = BlockKriging(K, H, W, f, k=2, halo_width=4, fit=False)
    out, _ = bk.run(torch.from_numpy(ks).cuda(), models=[VariogramModel("exponential", 0, 1, 4)] * 8)
    bk.finish()
    assert torch.all(out == 7.0)
    # tiling map: the merged volume at each (y, x) comes from the owning tile
    ids = np.zeros((K, H, W), np.float32)
    for b in bk.blocks:
        y0, y1, x0, x1 = b.core
        ids[:, y0:y1, x0:x1] = b.quadrant
    out, _ = bk.run(torch.from_numpy(ids).cuda(), models=[VariogramModel("exponential", 0, 1, 4)] * 8)
    bk.finish()
    o = out.cpu().numpy()
    for b in bk.blocks:
        y0, y1, x0, x1 = b.core
        # cores away from the seam: every plane equals the tile id
        assert np.all(o[:, y0 + 2:y1 - 2, x0 + 2:x1 - 2] == b.quadrant)
