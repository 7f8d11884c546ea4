"""Block partition -> per-block kriging -> merge: the reference's
``block_pipeline`` (absent from its code, SURVEY.md §8f
rank 2) on the device.

* ``partition`` tiles the slice plane into ``tiles_y x tiles_x`` in-plane
  blocks (the paper's 4 quadrants by default) and the stack
  into ``k`` Z chunks (n/k slices, the last chunk absorbs the remainder,
  SPEC.md:426).  Each block borrows ``halo_width`` voxels of known data from
  its neighbours on internal in-plane sides (border sides are not extended,
  SPEC.md:393, 422-424) and the next chunk's first slice in z (the trailing
  one-slice halo of the Z sub-part convention).
* ``BlockKriging`` runs one device plan per in-plane tile whose Z sub-parts
  are the chunks: every block fits its own variogram on its known voxels and
  fills its missing planes with its own clamp range (``reconstruct_block``'s
  kriging half); edge preservation stays reference host code
  (north_star).
* ``merge`` writes each output voxel from exactly one block's core region
  and discards the halos.  Blocks are value-independent,
  so the result does not depend on how they are scheduled.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .block_pipeline import ZPartKriging, output_depth, subpart_ranges
from .errors import TooFewSlices
from .kriging import _torch


@dataclass(frozen=True)
class BlockDescriptor:
    """One block: in-plane tile (ty, tx) and Z chunk c.  ``core`` is the
    region the block owns in the merged volume (y0, y1, x0, x1, exclusive
    ends), ``box`` the region it reads (core + halo), ``known`` the inclusive
    range of known slices it holds (trailing halo slice included)."""
    tile: tuple[int, int]
    chunk: int
    core: tuple[int, int, int, int]
    box: tuple[int, int, int, int]
    known: tuple[int, int]

    @property
    def quadrant(self) -> int:
        return self.tile[0] * 2 + self.tile[1]


def _split(n: int, parts: int) -> list[tuple[int, int]]:
    q = n // parts
    return [(i * q, (i + 1) * q if i < parts - 1 else n) for i in range(parts)]


def partition(n_known: int, height: int, width: int, k: int, halo_width: int = 2,
              tiles: tuple[int, int] = (2, 2)) -> list[BlockDescriptor]:
    """Descriptors of the ``tiles_y * tiles_x * k`` blocks in (tile, chunk)
    order."""
    ty_n, tx_n = tiles
    if k < 1 or ty_n < 1 or tx_n < 1 or halo_width < 0:
        raise ValueError("k, tiles must be >= 1 and halo_width >= 0")
    if height % ty_n or width % tx_n:
        raise ValueError(f"slice dims {height}x{width} must divide into {ty_n}x{tx_n} tiles")
    if n_known // k < 1 or n_known < 2 * k:
        raise TooFewSlices(f"{n_known} slices cannot form {k} chunks of >= 2 slices")
    chunks = subpart_ranges(n_known, k)
    out = []
    for iy, (y0, y1) in enumerate(_split(height, ty_n)):
        for ix, (x0, x1) in enumerate(_split(width, tx_n)):
            by0, by1 = (y0 - halo_width if iy > 0 else y0), (y1 + halo_width if iy < ty_n - 1 else y1)
            bx0, bx1 = (x0 - halo_width if ix > 0 else x0), (x1 + halo_width if ix < tx_n - 1 else x1)
            box = (max(0, by0), min(height, by1), max(0, bx0), min(width, bx1))
            for c, (b, e) in enumerate(chunks):
                out.append(BlockDescriptor((iy, ix), c, (y0, y1, x0, x1), box, (b, e)))
    return out


def check_tiling(blocks: list[BlockDescriptor], height: int, width: int) -> None:
    """Every (y, x) owned by exactly one tile core (TilingGap / TilingOverlap,
    SPEC.md:413)."""
    own = np.zeros((height, width), np.int32)
    for d in blocks:
        if d.chunk == 0:
            y0, y1, x0, x1 = d.core
            own[y0:y1, x0:x1] += 1
    if (own == 0).any():
        raise AssertionError("TilingGap: a voxel is owned by no block")
    if (own > 1).any():
        raise AssertionError("TilingOverlap: a voxel is owned by two blocks")


class BlockKriging:
    """Device block pipeline: partition -> per-block fit + fill -> merge.

    ``run(known)`` (device f32 [K, H, W]) returns the merged f32 volume
    [T, H, W] (and f64 variance when asked); ``finish()`` returns the
    per-block models in (tile, chunk) order.
    """

    def __init__(self, n_known: int, height: int, width: int, factor: int, k: int = 2,
                 halo_width: int = 2, tiles: tuple[int, int] = (2, 2), **kriging_kw):
        self.blocks = partition(n_known, height, width, k, halo_width, tiles)
        check_tiling(self.blocks, height, width)
        self.n_known, self.height, self.width, self.factor, self.k = n_known, height, width, factor, k
        self.depth = output_depth(n_known, factor)
        self.tiles = sorted({d.tile for d in self.blocks})
        self._plans = {}
        for t in self.tiles:
            d = next(b for b in self.blocks if b.tile == t)
            y0, y1, x0, x1 = d.box
            self._plans[t] = ZPartKriging(n_known, y1 - y0, x1 - x0, factor, k, **kriging_kw)

    def run(self, known, out=None, var=None, return_variance: bool = False, models=None):
        torch = _torch()
        if out is None:
            out = torch.empty((self.depth, self.height, self.width), dtype=torch.float32,
                              device=known.device)
        if return_variance and var is None:
            var = torch.empty((self.depth, self.height, self.width), dtype=torch.float64,
                              device=known.device)
        for t in self.tiles:
            d = next(b for b in self.blocks if b.tile == t)
            by0, by1, bx0, bx1 = d.box
            y0, y1, x0, x1 = d.core
            sub = known[:, by0:by1, bx0:bx1].contiguous()
            m = None
            if models is not None:
                m = [models[i] for i, b in enumerate(self.blocks) if b.tile == t]
            zk = self._plans[t]
            o, v = zk.run(sub, return_variance=var is not None, models=m)
            # merge: the tile's core, halos discarded
            out[:, y0:y1, x0:x1] = o[:, y0 - by0:y1 - by0, x0 - bx0:x1 - bx0]
            if var is not None:
                var[:, y0:y1, x0:x1] = v[:, y0 - by0:y1 - by0, x0 - bx0:x1 - bx0]
        return out, var

    def finish(self):
        """Per-block (model, (lo, hi)) in (tile, chunk) order; raises the
        reference's errors tagged with the failing block."""
        models, ranges = [], []
        for t in self.tiles:
            try:
                m, lohi = self._plans[t].finish()
            except Exception as exc:                       # SPEC.md:404 block identity
                raise type(exc)(f"block tile={t}: {exc}") from exc
            models.extend(m)
            ranges.extend([tuple(r) for r in np.asarray(lohi)])
        return models, ranges


def reconstruct_blocks(slices, factor: int, k: int = 2, halo_width: int = 2,
                       tiles: tuple[int, int] = (2, 2), return_variance: bool = False, **kw):
    """numpy in -> numpy out convenience wrapper of ``BlockKriging``."""
    torch = _torch()
    s = np.ascontiguousarray(slices, dtype=np.float32)
    K, H, W = s.shape
    bk = BlockKriging(K, H, W, factor, k, halo_width, tiles, **kw)
    out, var = bk.run(torch.from_numpy(s).cuda(), return_variance=return_variance)
    models, _ = bk.finish()
    return out.cpu().numpy(), (var.cpu().numpy() if var is not None else None), models
