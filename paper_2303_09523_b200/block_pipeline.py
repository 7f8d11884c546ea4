"""Z sub-part kriging pipeline: the kriging half of ``reconstruct_block``.

The reference's caller (``block_pipeline``: partition -> run_parallel ->
reconstruct_block -> merge) is absent from its code; the
paper splits the slice stack into equal Z sub-parts processed on separate
cores.  Here every sub-part is one unit of a single device
plan: each part fits its own variogram on its known voxels and fills its
missing planes with its own clamp range, exactly as a per-part
``fit_variogram`` + ``fill_missing``:

* part s holds known slices [s*q, (s+1)*q] (q = K // S; trailing one-slice
  halo; the remainder goes to the last part), placed at
  z = i*f in the part's grid;
* samples are the part's known voxels in ``np.nonzero`` order with (x, y, z)
  coordinates; ``fit_variogram(seed=0)`` defaults;
* the merged volume drops each part's trailing halo plane (the halo is a
  known plane, identical in both parts).

Across GPUs the parts are sharded contiguously (``zshard``); a rank needs the
first known slice of the next rank as its halo.
"""

from __future__ import annotations

import numpy as np

from .errors import TooFewSlices
from .kriging import KrigingPlan, VariogramModel, _torch


def subpart_ranges(n_known: int, n_subparts: int, part_len: int = 0) -> list[tuple[int, int]]:
    """Known-slice index ranges [b, e] of each part (inclusive halo)."""
    q = part_len or n_known // n_subparts
    if q < 1 or n_known < 2 or (n_subparts - 1) * q > n_known - 1:
        raise TooFewSlices(f"{n_known} slices cannot form {n_subparts} sub-parts")
    out = []
    for s in range(n_subparts):
        b = s * q
        e = (s + 1) * q if s < n_subparts - 1 else n_known - 1
        out.append((b, e))
    return out


def output_depth(n_known: int, factor: int) -> int:
    return n_known + (n_known - 1) * (factor - 1)


class ZPartKriging:
    """Device kriging path over the Z sub-parts of a regularly spaced stack.

    ``run(known)`` launches stats -> pair table -> bins -> fit -> solve ->
    predict on the current CUDA stream (asynchronous); ``finish()`` waits and
    returns the per-part ``VariogramModel`` list (raising the reference's
    errors, tagged with the failing part).  With ``fit=False`` the caller
    supplies one model per part and only stats -> solve -> predict run.
    """

    def __init__(self, n_known: int, height: int, width: int, factor: int,
                 n_subparts: int, kind: str = "exponential", drift: str = "linear",
                 accum: str = "fp64", n_bins: int = 15, max_pairs: int = 100_000,
                 seed: int = 0, force_generic: bool = False, fit: bool = True,
                 redraw_pairs: bool = False, part_len: int = 0, overlap: bool = True):
        if factor < 1:
            raise ValueError("factor must be >= 1")
        self.ranges = subpart_ranges(n_known, n_subparts, part_len)   # validates
        self.n_known, self.height, self.width = n_known, height, width
        self.factor, self.n_subparts, self.kind = factor, n_subparts, kind
        self.fit = fit
        self.depth = output_depth(n_known, factor)
        self.plan = KrigingPlan(height, width, self.depth,
                                np.arange(n_known, dtype=np.int32) * factor,
                                n_subparts=n_subparts, kind=kind, drift=drift,
                                accum=accum, fit=fit, n_bins=n_bins,
                                max_pairs=max_pairs, seed=seed,
                                force_generic=force_generic,
                                redraw_pairs=redraw_pairs, part_len=part_len,
                                overlap=overlap)

    @property
    def interpolated_voxels(self) -> int:
        return (self.n_known - 1) * (self.factor - 1) * self.height * self.width

    def allocate(self, return_variance: bool = False):
        torch = _torch()
        out = torch.empty((self.depth, self.height, self.width), dtype=torch.float32,
                          device="cuda")
        var = (torch.empty((self.depth, self.height, self.width), dtype=torch.float64,
                           device="cuda") if return_variance else None)
        return out, var

    def run(self, known, out=None, var=None, return_variance: bool = False, stream=None,
            models=None):
        """Launch the path; ``models`` ([S] VariogramModel or [S,3] array) is
        required when the object was built with ``fit=False``."""
        if out is None:
            out, v2 = self.allocate(return_variance)
            var = v2 if var is None else var
        if models is not None and not isinstance(models, np.ndarray):
            models = np.array([[m.nugget, m.sill, m.range_len] for m in models])
        self.plan.execute(known, out, var, models=models, stream=stream)
        return out, var

    def download(self, out, known_host, out_host=None, stream=None):
        """Volume to host memory, known planes taken from the host input
        (``KrigingPlan.download``)."""
        return self.plan.download(out, known_host, out_host, stream)

    def finish(self, stream=None):
        models, lohi = self.plan.finish(stream)
        return [VariogramModel(self.kind, *map(float, m)) for m in models], lohi


def reconstruct_zparts(slices, factor: int, n_subparts: int, kind: str = "exponential",
                       drift: str = "linear", return_variance: bool = False,
                       accum: str = "fp64", seed: int = 0):
    """Host-facing convenience: known slices (numpy [K,H,W] or CUDA tensor)
    -> (volume, variance or None, models).  numpy in, numpy out."""
    torch = _torch()
    host = isinstance(slices, np.ndarray)
    if host:
        known_host = torch.from_numpy(np.ascontiguousarray(slices, dtype=np.float32))
        known = known_host.cuda()
    else:
        known = slices.to(torch.float32).contiguous()
    K, H, W = known.shape
    zk = ZPartKriging(K, H, W, factor, n_subparts, kind=kind, drift=drift, accum=accum,
                      seed=seed)
    out, var = zk.run(known, return_variance=return_variance)
    if host:
        # interpolated planes from the device, known planes from the input
        vol = zk.download(out, known_host)
        models, _ = zk.finish()
        return vol.numpy(), (var.cpu().numpy() if var is not None else None), models
    models, _ = zk.finish()
    return out, var, models
