"""Block partition geometry (host side) and the oracle's
block composition -- CPU only."""

import numpy as np
import pytest

from oracle import kriging_oracle as O


def test_spec_partition_examples():
    from paper_2303_09523_b200.blocks import partition
    from paper_2303_09523_b200.errors import TooFewSlices
    # 50 slices of 1024x1024, k=2 -> 8 blocks of 25 slices, 512x512 (+ halo)
    bl = partition(50, 1024, 1024, k=2, halo_width=2)
    assert len(bl) == 8
    assert [b.known for b in bl[:2]] == [(0, 25), (25, 49)]        # 25 slices + trailing halo
    for b in bl:
        y0, y1, x0, x1 = b.core
        assert (y1 - y0, x1 - x0) == (512, 512)
        by0, by1, bx0, bx1 = b.box
        assert (by1 - by0, bx1 - bx0) == (514, 514)               # one internal side per axis
    # an interior tile (halo on both sides): 516x516 as SPEC.md:393
    bl = partition(50, 2048, 2048, k=2, halo_width=2, tiles=(4, 4))
    inner = [b for b in bl if b.tile == (1, 2)][0]
    assert (inner.box[1] - inner.box[0], inner.box[3] - inner.box[2]) == (516, 516)
    with pytest.raises(TooFewSlices):
        partition(4, 64, 64, k=4)
    with pytest.raises(ValueError):
        partition(8, 63, 64, k=2)


@pytest.mark.parametrize("tiles", [(2, 2), (1, 3), (3, 2)])
def test_tiling_exclusive_and_complete(tiles):
    from paper_2303_09523_b200.blocks import check_tiling, partition
    H, W = 12 * tiles[0], 10 * tiles[1]
    bl = partition(9, H, W, k=3, halo_width=2, tiles=tiles)
    check_tiling(bl, H, W)
    assert len(bl) == tiles[0] * tiles[1] * 3
    assert [(b.tile, b.chunk) for b in bl] == sorted((b.tile, b.chunk) for b in bl)
    # boxes never leave the plane, halos only on internal sides
    for b in bl:
        by0, by1, bx0, bx1 = b.box
        y0, y1, x0, x1 = b.core
        assert 0 <= by0 <= y0 and y1 <= by1 <= H and 0 <= bx0 <= x0 and x1 <= bx1 <= W
        assert (by0 == y0) == (y0 == 0) and (by1 == y1) == (y1 == H)
    # oracle restatement agrees with the package geometry
    ob = O.block_boxes(H, W, 2, tiles)
    pk = [(b.core, b.box) for b in bl if b.chunk == 0]
    assert ob == pk


def test_oracle_blocks_single_tile_is_zparts():
    r = np.random.default_rng(0)
    ks = (r.normal(size=(7, 12, 16)).cumsum(1).cumsum(2) * 10 + 100).astype(np.float32)
    a, ma = O.reconstruct_blocks(ks, 2, k=2, halo_width=0, tiles=(1, 1))
    b, _, mb = O.reconstruct_zparts(ks, 2, 2)
    assert np.array_equal(a, b)
    assert [m.sill for m in ma] == [m.sill for m in mb]


def test_oracle_blocks_known_planes_and_core_ownership():
    r = np.random.default_rng(1)
    ks = (r.normal(size=(5, 16, 16)).cumsum(1).cumsum(2) * 10 + 100).astype(np.float32)
    models = [O.Model("exponential", 0.1, 50.0, 6.0)] * 8
    out, _ = O.reconstruct_blocks(ks, 3, k=2, halo_width=2, models=models)
    assert np.array_equal(out[::3], ks)
    assert np.isfinite(out).all()
