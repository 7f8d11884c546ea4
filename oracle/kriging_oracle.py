"""CPU oracle for the kriging interpolation path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*.  It restates, in numpy/scipy, the algorithm of
the reference's plane-structured kriging path (``volkrig.kriging``) so that
the B200 product can be compared against it on the GPU box, where the
reference itself is not available.  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it.
The product package (``paper_2303_09523_b200``) never imports it and has no
CPU fallback.

Pinning: the restatement is checked against golden vectors produced by the
live reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/volkrig`` in the build container) and, when the
reference is importable, against the reference directly
(``tests/test_oracle_golden.py``).  Every function cites the reference
``file:line`` it follows; paths are relative to
``/root/reference/pkg/src/volkrig``.

Third-party arithmetic on the path is the same as the reference's: numpy
2.3 (``linalg.solve`` -> LAPACK dgesv, ``linalg.lstsq``, ``random.default_rng``
-> PCG64) and scipy 1.18 ``optimize.least_squares(method="trf")``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.optimize

KINDS = ("exponential", "gaussian", "spherical")
CONSTRAINT_TOL = 1e-8          # kriging.py:41
Z_SCHEDULE = (4, 8, 16)        # kriging.py:447 (z extents of the plane window)


class OracleError(Exception):
    pass


class InsufficientSamples(OracleError):
    pass


class DegenerateLags(OracleError):
    pass


class SingularSystem(OracleError):
    pass


class NoKnownNeighbors(OracleError):
    pass


# --------------------------------------------------------------------------
# variogram model                                       kriging.py:44-84
# --------------------------------------------------------------------------

@dataclass
class Model:
    kind: str
    nugget: float
    sill: float
    range_len: float

    def __post_init__(self):                           # kriging.py:53-57
        if self.kind not in KINDS:
            raise ValueError(f"kind must be one of {KINDS}")
        if self.nugget < 0 or self.sill < self.nugget or self.range_len <= 0:
            raise ValueError("need 0 <= nugget <= sill and range_len > 0")

    def semivariance(self, h):
        """gamma(h), 0 at h == 0 -- kriging.py:59-72."""
        lag = np.asarray(h, dtype=np.float64)
        partial = self.sill - self.nugget
        if self.kind == "exponential":
            shape = 1.0 - np.exp(-3.0 * lag / self.range_len)
        elif self.kind == "gaussian":
            shape = 1.0 - np.exp(-3.0 * (lag / self.range_len) ** 2)
        else:
            t = np.minimum(lag / self.range_len, 1.0)
            shape = 1.5 * t - 0.5 * t ** 3
        return np.where(lag == 0.0, 0.0, self.nugget + partial * shape)

    def cov(self, h):
        """C(h) = sill - gamma(h); unit white noise if sill <= 0 --
        kriging.py:74-84."""
        lag = np.asarray(h, dtype=np.float64)
        if self.sill <= 0.0:
            return np.where(lag == 0.0, 1.0, 0.0)
        return self.sill - self.semivariance(lag)


# --------------------------------------------------------------------------
# extended (universal-kriging) system                  kriging.py:87-245
# --------------------------------------------------------------------------

def drift_columns(rel: np.ndarray, drift: str) -> np.ndarray:
    """Drift design matrix on target-relative coords -- kriging.py:87-106."""
    if drift == "linear":
        return np.column_stack([np.ones(len(rel)), rel[:, 0], rel[:, 1],
                                rel[:, 2]])
    if drift == "constant":
        return np.ones((len(rel), 1))
    raise ValueError(f"unknown drift {drift!r}")


def independent_drift(Q: np.ndarray) -> list[int]:
    """Greedy lstsq rank test of drift columns -- kriging.py:145-156."""
    kept = [0]
    for j in range(1, Q.shape[1]):
        basis = Q[:, kept]
        coef = np.linalg.lstsq(basis, Q[:, j], rcond=None)[0]
        r = Q[:, j] - basis @ coef
        if np.linalg.norm(r) > 1e-9 * (np.linalg.norm(Q[:, j]) + 1.0):
            kept.append(j)
    return kept


def assemble(rel, model: Model, drift: str = "linear"):
    """Block matrix [[C, Q], [Q^T, 0]] and rhs [c0, q0] -- kriging.py:159-197.

    Returns (A, b, n, Q, q0).
    """
    rel = np.asarray(rel, dtype=np.float64).reshape(-1, 3)
    if len(rel) == 0:
        raise NoKnownNeighbors("cannot build a system with zero neighbors")
    Q = drift_columns(rel, drift)
    q0 = drift_columns(np.zeros((1, 3)), drift).reshape(-1)
    cols = independent_drift(Q)
    Q, q0 = Q[:, cols], q0[cols]
    delta = rel[:, None, :] - rel[None, :, :]
    C = model.cov(np.sqrt(np.sum(delta * delta, axis=-1)))
    c0 = model.cov(np.sqrt(np.sum(rel * rel, axis=-1)))
    n, p = len(rel), Q.shape[1]
    A = np.zeros((n + p, n + p))
    A[:n, :n] = C
    A[:n, n:] = Q
    A[n:, :n] = Q.T
    return A, np.concatenate([c0, q0]), n, Q, q0


def _try_solve(A, b):
    try:
        x = np.linalg.solve(A, b)
    except np.linalg.LinAlgError:
        return None
    return x if np.isfinite(x).all() else None


def solve(A, b, n, Q, q0):
    """LU solve, unbiasedness check, one ridge retry, kriging variance --
    kriging.py:200-245.  Returns (weights, lagrange, variance, ridged)."""
    def violated(x):
        r = Q.T @ x[:n] - q0
        return (float(np.max(np.abs(r))) if len(r) else 0.0) > CONSTRAINT_TOL

    x = _try_solve(A, b)
    ridged = False
    if x is None or violated(x):
        ridged = True
        ridge = max(1e-10 * np.trace(A[:n, :n]) / n, 1e-12)
        A2 = A.copy()
        A2[:n, :n] += ridge * np.eye(n)
        x = _try_solve(A2, b)
        if x is None:
            raise SingularSystem("extended kriging matrix is singular")
        if violated(x):
            raise SingularSystem("unbiasedness constraints unsatisfiable")
    w, lam = x[:n], x[n:]
    var = float(float(A[0, 0]) - w @ b[:n] - lam @ b[n:])
    return w, lam, var, ridged


def stencil_weights(rel, model: Model, drift: str = "linear"):
    """(weights, variance) for one relative-offset stencil -- the body of
    ``_WeightCache.weights_for`` (kriging.py:372-381)."""
    w, _, var, _ = solve(*assemble(rel, model, drift))
    return w, var


# --------------------------------------------------------------------------
# empirical semivariogram + bounded TRF fit            kriging.py:251-328
# --------------------------------------------------------------------------

def as_arrays(samples):
    """kriging.py:251-261."""
    if isinstance(samples, tuple) and len(samples) == 2:
        c = np.asarray(samples[0], dtype=np.float64).reshape(-1, 3)
        v = np.asarray(samples[1], dtype=np.float64).reshape(-1)
    else:
        c = np.asarray([s[0] for s in samples], dtype=np.float64)
        v = np.asarray([s[1] for s in samples], dtype=np.float64)
    if len(c) != len(v):
        raise ValueError("coords and values must align")
    return c, v


def pair_indices(m: int, max_pairs: int, seed: int):
    """Sample pairs exactly as kriging.py:278-286 (triu order when all pairs
    fit, else two PCG64 ``integers`` draws with i == j dropped)."""
    if m * (m - 1) // 2 <= max_pairs:
        return np.triu_indices(m, k=1)
    gen = np.random.default_rng(seed)
    i = gen.integers(0, m, size=max_pairs)
    j = gen.integers(0, m, size=max_pairs)
    ok = i != j
    return i[ok], j[ok]


@dataclass
class Bins:
    """Everything the fit needs -- kriging.py:288-309."""
    counts: np.ndarray      # per bin (all n_bins)
    sums: np.ndarray        # per bin sum of 0.5*dv^2 (all n_bins)
    hmax: float
    svar: float
    lag_max: float          # max over all kept pairs (constant-field model)
    edges: np.ndarray


def empirical_bins(coords, values, n_bins=15, max_pairs=100_000, seed=0):
    m = len(values)
    if m * (m - 1) // 2 < 30:                         # kriging.py:273-276
        raise InsufficientSamples(
            f"{m} samples give {m * (m - 1) // 2} pairs; need >= 30")
    i, j = pair_indices(m, max_pairs, seed)
    d = coords[i] - coords[j]
    lags = np.sqrt(np.sum(d * d, axis=-1))
    if not (lags > 0).any():                           # kriging.py:290-291
        raise DegenerateLags("all sample pairs are co-located")
    half_sq = 0.5 * (values[i] - values[j]) ** 2
    svar = float(values.var())
    lag_max = float(lags.max())
    pos = lags > 0
    lags, half_sq = lags[pos], half_sq[pos]
    hmax = float(lags.max())
    edges = np.linspace(0.0, hmax, n_bins + 1)
    b = np.clip(np.digitize(lags, edges) - 1, 0, n_bins - 1)
    counts = np.bincount(b, minlength=n_bins)
    sums = np.bincount(b, weights=half_sq, minlength=n_bins)
    return Bins(counts, sums, hmax, svar, lag_max, edges)


def fit_bins(bins: Bins, kind="exponential") -> Model:
    """Count-weighted bounded TRF fit of (nugget, psill, range) --
    kriging.py:294-328."""
    if bins.svar == 0.0:
        return Model(kind, 0.0, 0.0, max(bins.lag_max, 1.0))
    nz = bins.counts > 0
    centres = (0.5 * (bins.edges[:-1] + bins.edges[1:]))[nz]
    gamma_emp = bins.sums[nz] / bins.counts[nz]
    weight = np.sqrt(bins.counts[nz].astype(np.float64))

    def residual(p):
        nug = max(p[0], 0.0)
        mdl = Model(kind, nug, nug + max(p[1], 0.0), max(p[2], 1e-6))
        return weight * (mdl.semivariance(centres) - gamma_emp)

    svar, hmax = bins.svar, bins.hmax
    res = scipy.optimize.least_squares(
        residual, np.array([0.0, svar, hmax / 3.0]),
        bounds=([0.0, 0.0, 1e-6],
                [2.0 * svar + 1e-12, 4.0 * svar + 1e-12, 10.0 * hmax]),
        method="trf")
    nug = float(max(res.x[0], 0.0))
    return Model(kind, nug, nug + float(max(res.x[1], 0.0)),
                 float(max(res.x[2], 1e-6)))


def fit_variogram(samples, kind="exponential", n_bins=15, max_pairs=100_000,
                  seed=0) -> Model:
    """kriging.py:264-328."""
    c, v = as_arrays(samples)
    return fit_bins(empirical_bins(c, v, n_bins, max_pairs, seed), kind)


# --------------------------------------------------------------------------
# plane-structured fill                                kriging.py:334-557
# --------------------------------------------------------------------------

def window(c: int, extent: int, size: int) -> tuple[int, int]:
    """Half-open clamped window [c-(e/2-1), c+e/2] -- kriging.py:334-342."""
    return max(0, c - (extent // 2 - 1)), min(size, c + extent // 2 + 1)


def plane_window(z: int, known_z: np.ndarray, depth: int):
    """Known planes read by missing plane z (z-extent 4 -> 8 -> 16 until the
    set brackets z) -- kriging.py:444-455 with _bracketed at :360-361."""
    chosen = None
    for ext in Z_SCHEDULE:
        lo, hi = window(z, ext, depth)
        sel = known_z[(known_z >= lo) & (known_z < hi)]
        if len(sel) == 0:
            continue
        chosen = sel
        if (sel < z).any() and (sel > z).any():
            break
    return chosen


def plane_flags(mask: np.ndarray):
    """Per-plane missing flags or None -- kriging.py:434-441."""
    flat = mask.reshape(mask.shape[0], -1)
    anym, allm = flat.any(axis=1), flat.all(axis=1)
    return anym if np.array_equal(anym, allm) else None


def fill_missing(data, mask, model: Model, drift="linear",
                 return_variance=False):
    """``fill_missing`` -- kriging.py:458-496: the plane-structured stencil
    path (kriging.py:499-557) or, for any other mask, the per-voxel window
    path (``fill_generic``, kriging.py:408-431).

    ``data`` float32 [dz, dy, dx] with NaN planes, ``mask`` bool.  Returns
    (out float32, var float64 or None).
    """
    data = np.ascontiguousarray(data, dtype=np.float32)
    mask = np.ascontiguousarray(mask, dtype=bool)
    if not np.array_equal(np.isnan(data), mask):            # model.py:111-117
        raise ValueError("missing_mask out of sync with NaN sentinel")
    if not np.isfinite(data[~mask]).all():
        raise ValueError("known voxels must be finite")
    if not mask.any():                                      # kriging.py:469-473
        return data.copy(), (np.zeros(data.shape) if return_variance else None)
    known = data[~mask]
    if known.size == 0:
        raise NoKnownNeighbors("grid has no known voxels at all")
    lo, hi = float(known.min()), float(known.max())
    out = data.copy()
    var = np.zeros(data.shape) if return_variance else None
    flags = plane_flags(mask)
    if flags is None:                                       # kriging.py:488-490
        return fill_generic(data, mask, model, drift, lo, hi, out, var)

    dz, dy, dx = data.shape
    known_z = np.nonzero(~flags)[0]
    cache: dict[bytes, tuple] = {}
    border_cache: dict[tuple, tuple] = {}

    def weights(rel):
        key = rel.astype(np.int16).tobytes()
        if key not in cache:
            cache[key] = stencil_weights(rel, model, drift)
        return cache[key]

    for z in np.nonzero(flags)[0]:
        z = int(z)
        planes = plane_window(z, known_z, dz)
        if planes is None:
            raise NoKnownNeighbors(f"no known plane within reach of z={z}")
        offs = [int(p) - z for p in planes]
        interior = dx >= 4 and dy >= 4
        if interior:                                        # kriging.py:517-530
            rel = np.array([(ox, oy, oz) for oz in offs
                            for oy in range(-1, 3) for ox in range(-1, 3)],
                           dtype=np.int64)
            w, v = weights(rel)
            acc = np.zeros((dy - 3, dx - 3))
            for t in range(len(w)):
                ox, oy, oz = rel[t]
                acc += w[t] * data[z + oz, 1 + oy:dy - 2 + oy,
                                   1 + ox:dx - 2 + ox]
            np.clip(acc, lo, hi, out=acc)
            out[z, 1:dy - 2, 1:dx - 2] = acc
            if var is not None:
                var[z, 1:dy - 2, 1:dx - 2] = v
            border = [(y, x) for y in range(dy) for x in range(dx)
                      if not (1 <= y <= dy - 3 and 1 <= x <= dx - 3)]
        else:
            border = [(y, x) for y in range(dy) for x in range(dx)]
        # border voxels, clamped windows -- kriging.py:531-557: the solved
        # stencil of each (plane offsets, clamped window) is looked up by that
        # key, as the reference's border_cache does (the same weights as a
        # rebuilt offset list: the key determines the list)
        dz_key = tuple(offs)
        for (y, x) in border:
            xlo, xhi = window(x, 4, dx)
            ylo, yhi = window(y, 4, dy)
            key = (dz_key, xlo - x, xhi - x, ylo - y, yhi - y)
            hit = border_cache.get(key)
            if hit is None:
                rel = np.array([(ox - x, oy - y, oz) for oz in offs
                                for oy in range(ylo, yhi)
                                for ox in range(xlo, xhi)], dtype=np.int64)
                hit = weights(rel)
                border_cache[key] = hit
            w, v = hit
            vals = np.concatenate([data[z + oz, ylo:yhi, xlo:xhi].ravel()
                                   for oz in offs])
            pred = float(w @ vals)
            out[z, y, x] = min(max(pred, lo), hi)
            if var is not None:
                var[z, y, x] = v
    return out, var


# --------------------------------------------------------------------------
# generic per-voxel path                               kriging.py:37-40, 345-431
# --------------------------------------------------------------------------

WINDOW_SCHEDULE = ((4, 4), (4, 8), (4, 16), (8, 16), (16, 16))   # kriging.py:39


def gather_window(mask, x, y, z, inplane, z_extent):
    """Known voxels of the clamped window around (x, y, z) in np.nonzero
    (z, y, x) order, as (x, y, z) coords -- kriging.py:345-357."""
    dz, dy, dx = mask.shape
    x0, x1 = window(x, inplane, dx)
    y0, y1 = window(y, inplane, dy)
    z0, z1 = window(z, z_extent, dz)
    kz, ky, kx = np.nonzero(~mask[z0:z1, y0:y1, x0:x1])
    if len(kz) == 0:
        return None
    return np.column_stack([kx + x0, ky + y0, kz + z0])


def choose_window(mask, x, y, z):
    """The schedule walk of ``_predict_generic`` -- kriging.py:414-424: the
    first window whose known voxels bracket z, or at z extent 16 the first
    window with any known voxel.  Returns (schedule index, coords) or None."""
    for i, (inplane, z_extent) in enumerate(WINDOW_SCHEDULE):
        coords = gather_window(mask, x, y, z, inplane, z_extent)
        if coords is None:
            continue
        cz = coords[:, 2]
        if ((cz < z).any() and (cz > z).any()) or z_extent == 16:
            return i, coords
    return None


def fill_generic(data, mask, model: Model, drift, lo, hi, out, var):
    """Per-voxel path over np.argwhere(mask) raster order, weights cached by
    the int16 relative-offset signature -- kriging.py:408-431, 364-381."""
    cache: dict[bytes, tuple] = {}
    for z, y, x in np.argwhere(mask):
        got = choose_window(mask, int(x), int(y), int(z))
        if got is None:
            raise NoKnownNeighbors(f"no known voxel near {(int(x), int(y), int(z))}")
        coords = got[1]
        rel = coords - np.array([x, y, z])
        key = rel.astype(np.int16).tobytes()
        if key not in cache:
            cache[key] = stencil_weights(rel, model, drift)
        w, v = cache[key]
        vals = data[coords[:, 2], coords[:, 1], coords[:, 0]].astype(np.float64)
        pred = float(w @ vals)
        out[z, y, x] = min(max(pred, lo), hi)
        if var is not None:
            var[z, y, x] = v
    return out, var


# --------------------------------------------------------------------------
# Z sub-part pipeline (SPEC.md:392-427 partition/merge)
# --------------------------------------------------------------------------

def missing_planes_per_gap(gap_mm: float, spacing_mm: float) -> int:
    """model.py:205-217."""
    if gap_mm <= 0 or spacing_mm <= 0:
        raise ValueError("gap and spacing must be > 0")
    return max(0, int(np.floor(gap_mm / spacing_mm + 0.5)) - 1)


def subpart_ranges(n_known: int, n_parts: int):
    """Known-slice index ranges [b, e] (inclusive, trailing one-slice halo)
    of each Z sub-part; the remainder goes to the last part."""
    q = n_known // n_parts
    if q < 1:
        raise ValueError("more sub-parts than known slices")
    out = []
    for s in range(n_parts):
        b = s * q
        e = (s + 1) * q if s < n_parts - 1 else n_known - 1
        out.append((b, e))
    return out


def subpart_grid(slices, b, e, factor):
    """NaN grid of one sub-part with known slice i at z = (i-b)*factor."""
    nk = e - b + 1
    h, w = slices.shape[1:]
    depth = (nk - 1) * factor + 1
    data = np.full((depth, h, w), np.nan, dtype=np.float32)
    data[::factor] = slices[b:e + 1]
    return data, np.isnan(data)


def subpart_samples(data, mask):
    """Known voxels in np.nonzero order with (x, y, z) coords -- the sample
    convention of kriging.py:354-356 applied to a whole sub-part."""
    kz, ky, kx = np.nonzero(~mask)
    coords = np.column_stack([kx, ky, kz]).astype(np.float64)
    return coords, data[kz, ky, kx].astype(np.float64)


def reconstruct_zpart(slices, b, e, factor, kind="exponential",
                      drift="linear", return_variance=False, seed=0):
    """``reconstruct_block`` kriging half for one Z sub-part:
    fit_variogram on the sub-part's known voxels, then fill_missing."""
    data, mask = subpart_grid(slices, b, e, factor)
    model = fit_variogram(subpart_samples(data, mask), kind, seed=seed)
    out, var = fill_missing(data, mask, model, drift, return_variance)
    return out, var, model


def reconstruct_zparts(slices, factor, n_parts, kind="exponential",
                       drift="linear", return_variance=False, seed=0):
    """Partition -> per-part fit+fill -> merge by dropping each part's
    trailing halo plane.  Returns (volume, variance or None, models)."""
    slices = np.ascontiguousarray(slices, dtype=np.float32)
    k = slices.shape[0]
    depth = (k - 1) * factor + 1
    vol = np.empty((depth,) + slices.shape[1:], dtype=np.float32)
    var = np.zeros(vol.shape) if return_variance else None
    models = []
    for (b, e) in subpart_ranges(k, n_parts):
        out, v, mdl = reconstruct_zpart(slices, b, e, factor, kind, drift,
                                        return_variance, seed)
        z0 = b * factor
        vol[z0:z0 + out.shape[0]] = out
        if var is not None:
            var[z0:z0 + out.shape[0]] = v
        models.append(mdl)
    return vol, var, models


def interpolated_voxels(n_known: int, factor: int, h: int, w: int) -> int:
    return (n_known - 1) * (factor - 1) * h * w


# --------------------------------------------------------------------------
# block pipeline (absent from the reference's code)
# --------------------------------------------------------------------------

def block_boxes(height, width, halo_width=2, tiles=(2, 2)):
    """In-plane tiles: (core, box) with the halo on internal sides only --
    SPEC.md:388-395, 422-424."""
    ty_n, tx_n = tiles
    ys = [(i * (height // ty_n), (i + 1) * (height // ty_n) if i < ty_n - 1 else height)
          for i in range(ty_n)]
    xs = [(i * (width // tx_n), (i + 1) * (width // tx_n) if i < tx_n - 1 else width)
          for i in range(tx_n)]
    out = []
    for iy, (y0, y1) in enumerate(ys):
        for ix, (x0, x1) in enumerate(xs):
            by0 = y0 - halo_width if iy > 0 else y0
            by1 = y1 + halo_width if iy < ty_n - 1 else y1
            bx0 = x0 - halo_width if ix > 0 else x0
            bx1 = x1 + halo_width if ix < tx_n - 1 else x1
            out.append(((y0, y1, x0, x1), (max(0, by0), min(height, by1), max(0, bx0), min(width, bx1))))
    return out


def reconstruct_blocks(slices, factor, k=2, halo_width=2, tiles=(2, 2), models=None):
    """partition -> per-block fit + fill -> merge: every
    in-plane tile runs the Z sub-part pipeline with k chunks; the merged
    volume keeps each tile's core.  ``models`` ([tiles*k] Model, (tile,
    chunk) order) skips the fits."""
    slices = np.ascontiguousarray(slices, dtype=np.float32)
    K, H, W = slices.shape
    T = K + (K - 1) * (factor - 1)
    out = np.empty((T, H, W), np.float32)
    all_models = []
    for ti, ((y0, y1, x0, x1), (by0, by1, bx0, bx1)) in enumerate(block_boxes(H, W, halo_width, tiles)):
        sub = slices[:, by0:by1, bx0:bx1]
        if models is None:
            vol, _, ms = reconstruct_zparts(sub, factor, k)
        else:
            ms = models[ti * k:(ti + 1) * k]
            vol = np.empty((T, by1 - by0, bx1 - bx0), np.float32)
            for c, (b, e) in enumerate(subpart_ranges(K, k)):
                d, m = subpart_grid(sub, b, e, factor)
                o, _ = fill_missing(d, m, ms[c])
                vol[b * factor:b * factor + o.shape[0]] = o
        out[:, y0:y1, x0:x1] = vol[:, y0 - by0:y1 - by0, x0 - bx0:x1 - bx0]
        all_models.extend(ms)
    return out, all_models

