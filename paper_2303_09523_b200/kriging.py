"""Drop-in kriging entry points backed by the sm_100a kernels.

Mirrors the reference's public API (``volkrig.kriging``):

* ``VariogramModel``                       kriging.py:44-84
* ``fit_variogram(samples, kind, n_bins, max_pairs, seed)``   kriging.py:264-328
* ``fill_missing(grid, model, drift, return_variance)``       kriging.py:458-557

with the same argument meaning, return types and exception classes.  The
numerics run on the GPU through the C ABI in ``include/volkrig_b200.h``; there
is no CPU fallback -- without a CUDA device or the built library these raise.
One optional keyword is added: ``accum`` ("fp64" default, as the reference;
"fp32" accumulates the prediction stencil in fp32; "fixed" runs it as exact
integer tensor-core products of 24-bit fixed-point values and 32-bit
fixed-point weights, error <= ~2e-7 of the data range; solves stay fp64).
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import (DeviceError, DeviceUnsupported, InsufficientSamples,
                     NoKnownNeighbors, raise_for_status)
from .model import VolumeGrid

VARIOGRAM_KINDS = ("exponential", "gaussian", "spherical")
WPAD = 128


@dataclass
class VariogramModel:
    """Isotropic variogram nugget + (sill - nugget) * shape(h / range_len)."""

    kind: str
    nugget: float
    sill: float
    range_len: float

    def __post_init__(self):
        if self.kind not in VARIOGRAM_KINDS:
            raise ValueError(f"kind must be one of {VARIOGRAM_KINDS}")
        if self.nugget < 0 or self.sill < self.nugget or self.range_len <= 0:
            raise ValueError("need 0 <= nugget <= sill and range_len > 0")

    def gamma(self, h):
        h = np.asarray(h, dtype=np.float64)
        ps, r = self.sill - self.nugget, self.range_len
        if self.kind == "exponential":
            shape = 1.0 - np.exp(-3.0 * h / r)
        elif self.kind == "gaussian":
            shape = 1.0 - np.exp(-3.0 * (h / r) ** 2)
        else:
            t = np.minimum(h / r, 1.0)
            shape = 1.5 * t - 0.5 * t ** 3
        return np.where(h == 0.0, 0.0, self.nugget + ps * shape)

    def covariance(self, h):
        h = np.asarray(h, dtype=np.float64)
        if self.sill <= 0.0:
            return np.where(h == 0.0, 1.0, 0.0)
        return self.sill - self.gamma(h)

    def as_array(self) -> np.ndarray:
        return np.array([self.nugget, self.sill, self.range_len], dtype=np.float64)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required (no CPU fallback)")
    return torch


def _stream_handle(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _upload(arr: np.ndarray):
    """A device copy of a host numpy array through the library's staged
    uploader (``vk_copy_h2d``: page-locked chunks filled by host threads while
    the previous chunk's DMA runs), on torch's current stream."""
    torch = _torch()
    arr = np.ascontiguousarray(arr)
    dt = torch.from_numpy(arr[:0]).dtype
    out = torch.empty(arr.shape, dtype=dt, device="cuda")
    if arr.nbytes:
        raise_for_status(_lib.load().vk_copy_h2d(out.data_ptr(), arr.ctypes.data, arr.nbytes,
                                                 _stream_handle(None)))
    return out


def _model_params(model):
    """(kind, [nugget, sill, range_len]) of any object with the reference
    VariogramModel's attributes (kriging.py:44-57) -- ours or volkrig's."""
    kind = model.kind
    if kind not in VARIOGRAM_KINDS:
        raise ValueError(f"kind must be one of {VARIOGRAM_KINDS}")
    return kind, np.array([float(model.nugget), float(model.sill), float(model.range_len)],
                          dtype=np.float64)


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and bool(x.is_cuda)


def _grid_parts(grid):
    """(data, mask, origin_offset, on_device) of any object with the reference
    VolumeGrid's attributes (model.py:71-92): ``.data`` [z, y, x],
    ``.missing_mask`` (None -> NaN sentinel), ``.origin_offset``."""
    data = grid.data
    mask = getattr(grid, "missing_mask", None)
    origin = tuple(getattr(grid, "origin_offset", (0, 0, 0)))
    on_dev = _is_cuda_tensor(data)
    if on_dev:
        torch = _torch()
        data = data.to(torch.float32).contiguous()
        mask = (torch.isnan(data) if mask is None else mask.to(torch.bool)).contiguous()
    else:
        data = np.ascontiguousarray(data, dtype=np.float32)
        mask = np.ascontiguousarray(np.isnan(data) if mask is None else mask, dtype=bool)
    if tuple(mask.shape) != tuple(data.shape) or len(data.shape) != 3:
        raise ValueError("volume data must be 3D with a mask of the same shape")
    return data, mask, origin, on_dev


def _like_grid(grid, data, mask, origin):
    """A result grid of the caller's grid type (the reference's VolumeGrid for
    a reference grid), falling back to ours for device data."""
    cls = type(grid)
    if cls is not VolumeGrid:
        try:
            return cls(data, mask, origin)
        except Exception:
            pass
    return VolumeGrid(data, mask, origin)


class KrigingPlan:
    """A device plan: geometry tables, stencil systems and workspace for one
    grid layout (``vk_plan``).  ``execute`` is stream-ordered and async;
    ``finish`` synchronises and raises the reference's exceptions."""

    def __init__(self, height, width, depth, known_z, n_subparts=1,
                 kind="exponential", drift="linear", accum="fp64", fit=True,
                 n_bins=15, max_pairs=100_000, seed=0, force_generic=False,
                 part_len=0, redraw_pairs=False, overlap=True):
        if callable(drift):
            raise DeviceUnsupported("a callable drift cannot cross the C ABI; "
                                    "use 'linear' or 'constant'")
        if drift not in _lib.DRIFT_IDS:
            raise ValueError(f"unknown drift {drift!r}")
        if kind not in _lib.KIND_IDS:
            raise ValueError(f"kind must be one of {VARIOGRAM_KINDS}")
        if accum not in _lib.ACCUM_IDS:
            raise ValueError("accum must be 'fp64', 'fp32' or 'fixed'")
        _torch()
        self.lib = _lib.load()
        kz = np.ascontiguousarray(known_z, dtype=np.int32)
        self._kz = kz
        self.height, self.width, self.depth = int(height), int(width), int(depth)
        self.n_known = len(kz)
        self.n_subparts = int(n_subparts)
        self.kind, self.drift, self.accum, self.fit = kind, drift, accum, bool(fit)
        desc = _lib.PlanDesc(
            self.height, self.width, self.depth, len(kz),
            kz.ctypes.data_as(C.POINTER(C.c_int32)), self.n_subparts,
            _lib.KIND_IDS[kind], _lib.DRIFT_IDS[drift], _lib.ACCUM_IDS[accum],
            int(n_bins), int(max_pairs), int(seed), int(bool(fit)),
            (_lib.FLAG_FORCE_GENERIC if force_generic else 0)
            | (_lib.FLAG_REDRAW_PAIRS if redraw_pairs else 0)
            | (0 if overlap else _lib.FLAG_SERIAL), int(part_len))
        handle = C.c_void_p()
        raise_for_status(self.lib.vk_plan_create(C.byref(desc), C.byref(handle)))
        self._h = handle
        self._info = None

    # -- introspection ------------------------------------------------------
    @property
    def info(self) -> dict:
        inf = _lib.PlanInfo()
        raise_for_status(self.lib.vk_plan_get_info(self._h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in _lib.PlanInfo._fields_}

    @property
    def interpolated_voxels(self) -> int:
        return int(self.info["interpolated_voxels"])

    # -- execution ------------------------------------------------------------
    def execute(self, known, out, var=None, models=None, stream=None) -> None:
        torch = _torch()
        K, H, W = self.n_known, self.height, self.width
        if not (known.is_cuda and known.dtype == torch.float32 and known.is_contiguous()
                and tuple(known.shape) == (K, H, W)):
            raise ValueError(f"known must be a contiguous CUDA float32 [{K},{H},{W}] tensor")
        if not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()
                and tuple(out.shape) == (self.depth, H, W)):
            raise ValueError("out must be a contiguous CUDA float32 [depth,H,W] tensor")
        vptr = None
        if var is not None:
            if not (var.is_cuda and var.dtype == torch.float64 and var.is_contiguous()
                    and tuple(var.shape) == (self.depth, H, W)):
                raise ValueError("var must be a contiguous CUDA float64 [depth,H,W] tensor")
            vptr = var.data_ptr()
        mptr = None
        if not self.fit:
            if models is None:
                raise ValueError("models are required for a plan without fitting")
            self._models_in = np.ascontiguousarray(models, dtype=np.float64).reshape(
                self.n_subparts, 3)
            mptr = self._models_in.ctypes.data
        raise_for_status(self.lib.vk_plan_execute(
            self._h, known.data_ptr(), mptr, out.data_ptr(), vptr,
            _stream_handle(stream)))

    def download(self, out, known_host, out_host=None, stream=None):
        """Reconstructed volume -> host (``vk_plan_download``): interpolated
        planes from the device ``out``, known planes from the caller's host
        input ``known_host`` (CPU float32 [K,H,W]; pinned for overlap).
        Returns the host float32 [depth,H,W] tensor (pinned if allocated
        here).  Stream-ordered: synchronise before reading it."""
        torch = _torch()
        K, H, W = self.n_known, self.height, self.width
        if not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()
                and tuple(out.shape) == (self.depth, H, W)):
            raise ValueError("out must be a contiguous CUDA float32 [depth,H,W] tensor")
        if not (not known_host.is_cuda and known_host.dtype == torch.float32 and known_host.is_contiguous()
                and tuple(known_host.shape) == (K, H, W)):
            raise ValueError(f"known_host must be a contiguous CPU float32 [{K},{H},{W}] tensor")
        if out_host is None:
            out_host = torch.empty((self.depth, H, W), dtype=torch.float32, pin_memory=True)
        elif not (not out_host.is_cuda and out_host.dtype == torch.float32 and out_host.is_contiguous()
                  and tuple(out_host.shape) == (self.depth, H, W)):
            raise ValueError("out_host must be a contiguous CPU float32 [depth,H,W] tensor")
        raise_for_status(self.lib.vk_plan_download(self._h, out.data_ptr(), known_host.data_ptr(),
                                                   out_host.data_ptr(), _stream_handle(stream)))
        return out_host

    def finish(self, stream=None):
        """Synchronise; return (models [S,3], lohi [S,2]) or raise."""
        models = np.zeros((self.n_subparts, 3))
        lohi = np.zeros((self.n_subparts, 2))
        failed = C.c_int32(-1)
        code = self.lib.vk_plan_finish(self._h, _stream_handle(stream), C.byref(failed),
                                       models.ctypes.data, lohi.ctypes.data)
        ctx = f"sub-part {failed.value}" if failed.value >= 0 and self.n_subparts > 1 else ""
        raise_for_status(code, ctx)
        return models, lohi

    def set_timing(self, ring: int = 1) -> None:
        """Record per-stage CUDA events for the last ``ring`` executes."""
        raise_for_status(self.lib.vk_plan_set_timing(self._h, int(ring)))

    def stage_ms(self, back: int = 0) -> dict:
        """Per-stage device times (ms) of the execute ``back`` calls ago."""
        ms = np.zeros(_lib.N_STAGES, dtype=np.float32)
        raise_for_status(self.lib.vk_plan_stage_ms(self._h, int(back), ms.ctypes.data))
        return dict(zip(_lib.STAGES, map(float, ms)))

    def systems(self):
        """Solved stencils: (weights [n,128], variance [n], ids [n,4])."""
        n = self.info["n_systems"]
        w = np.zeros((n, WPAD))
        v = np.zeros(n)
        ids = np.zeros((n, 4), np.int32)
        raise_for_status(self.lib.vk_plan_get_systems(self._h, w.ctypes.data, v.ctypes.data,
                                                      ids.ctypes.data))
        return w, v, ids

    def close(self):
        if getattr(self, "_h", None):
            self.lib.vk_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_PLANS: "OrderedDict[tuple, KrigingPlan]" = OrderedDict()


def cached_plan(**kw) -> KrigingPlan:
    torch = _torch()
    key = tuple(sorted((k, tuple(v) if isinstance(v, (list, np.ndarray)) else v)
                       for k, v in kw.items())) + (torch.cuda.current_device(),)
    plan = _PLANS.get(key)
    if plan is None:
        plan = KrigingPlan(**kw)
        _PLANS[key] = plan
        while len(_PLANS) > 8:
            _PLANS.popitem(last=False)[1].close()
    else:
        _PLANS.move_to_end(key)
    return plan


# --------------------------------------------------------------------------
# fit_variogram                                          kriging.py:264-328
# --------------------------------------------------------------------------

def _as_coord_value_arrays(samples):
    if isinstance(samples, tuple) and len(samples) == 2:
        coords = np.asarray(samples[0], dtype=np.float64).reshape(-1, 3)
        values = np.asarray(samples[1], dtype=np.float64).reshape(-1)
    else:
        coords = np.asarray([s[0] for s in samples], dtype=np.float64)
        values = np.asarray([s[1] for s in samples], dtype=np.float64)
    if len(coords) != len(values):
        raise ValueError("coords and values must align")
    return coords, values


def fit_variogram(samples, kind: str = "exponential", n_bins: int = 15,
                  max_pairs: int = 100_000, seed: int = 0) -> VariogramModel:
    """Empirical semivariogram + bounded TRF fit, on the device."""
    if kind not in VARIOGRAM_KINDS:
        raise ValueError(f"kind must be one of {VARIOGRAM_KINDS}")
    coords, values = _as_coord_value_arrays(samples)
    m = len(values)
    if m * (m - 1) // 2 < 30:
        raise InsufficientSamples(f"{m} samples give {m * (m - 1) // 2} pairs; need >= 30")
    torch = _torch()
    lib = _lib.load()
    c_d = _upload(coords)
    v_d = _upload(values)
    out = np.zeros(3)
    raise_for_status(lib.vk_fit_variogram_samples(
        c_d.data_ptr(), v_d.data_ptr(), m, _lib.KIND_IDS[kind], int(n_bins),
        int(max_pairs), int(seed), out.ctypes.data, _stream_handle(None)))
    return VariogramModel(kind, float(out[0]), float(out[1]), float(out[2]))


# --------------------------------------------------------------------------
# fill_missing                                           kriging.py:458-557
# --------------------------------------------------------------------------

def _scan_grid(data_d, mask_d):
    """Device validate() + plane structure: per-plane (#missing, #nan,
    #nan != mask, #known non-finite)."""
    torch = _torch()
    lib = _lib.load()
    T = data_d.shape[0]
    P = data_d[0].numel()
    counts = torch.empty((T, 4), dtype=torch.int32, device=data_d.device)
    raise_for_status(lib.vk_grid_scan(data_d.data_ptr(), mask_d.data_ptr(), T, P,
                                      counts.data_ptr(), _stream_handle(None)))
    return counts.cpu().numpy()


def solve_systems(rels, model: VariogramModel, drift="linear"):
    """``build_system`` + ``solve_ked`` (kriging.py:159-245) for a batch of
    neighbour sets, on the device (``vk_solve_systems``).  ``rels`` is a list
    of (n_i, 3) integer target-relative (x, y, z) offsets; returns (list of
    weight arrays, variance array).  Raises ``SingularSystem`` like the
    reference when a system stays singular after the ridge retry."""
    torch = _torch()
    if callable(drift):
        raise DeviceUnsupported("a callable drift cannot cross the C ABI")
    if drift not in _lib.DRIFT_IDS:
        raise ValueError(f"unknown drift {drift!r}")
    arrs = [np.asarray(r, dtype=np.int64).reshape(-1, 3) for r in rels]
    if any(a.size and np.abs(a).max() > 32767 for a in arrs):
        raise ValueError("relative offsets must fit int16")
    off = np.zeros(len(arrs) + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in arrs])
    rel_d = torch.from_numpy(np.concatenate(arrs).astype(np.int16) if arrs else
                             np.zeros((0, 3), np.int16)).cuda()
    w_d = torch.empty(int(off[-1]), dtype=torch.float64, device="cuda")
    v_d = torch.empty(len(arrs), dtype=torch.float64, device="cuda")
    kind, m = _model_params(model)
    raise_for_status(_lib.load().vk_solve_systems(
        rel_d.data_ptr(), off.ctypes.data, len(arrs), _lib.KIND_IDS[kind],
        _lib.DRIFT_IDS[drift], m.ctypes.data, w_d.data_ptr(), v_d.data_ptr(), None,
        _stream_handle(None)))
    w = w_d.cpu().numpy()
    return [w[off[i]:off[i + 1]] for i in range(len(arrs))], v_d.cpu().numpy()


def interpolate_voxel(grid: VolumeGrid, target, model: VariogramModel, drift="linear",
                      inplane: int = 4, z_extent: int = 4,
                      clamp_range: tuple[float, float] | None = None) -> float:
    """kriging.py:384-405: one voxel from the known voxels of its
    (inplane, z_extent) window, clamped to the grid's known range.  The
    window gather is index arithmetic on the mask; the system is solved on
    the device (``solve_systems``)."""
    x, y, z = (int(v) for v in target)
    data, mask, _, on_dev = _grid_parts(grid)
    if on_dev:
        data, mask = data.cpu().numpy(), mask.cpu().numpy()
    if not mask[z, y, x]:
        return float(data[z, y, x])
    dz, dy, dx = data.shape

    def win(c, extent, size):                      # kriging.py:334-342
        return max(0, c - (extent // 2 - 1)), min(size, c + extent // 2 + 1)
    x0, x1 = win(x, inplane, dx)
    y0, y1 = win(y, inplane, dy)
    z0, z1 = win(z, z_extent, dz)
    kz, ky, kx = np.nonzero(~mask[z0:z1, y0:y1, x0:x1])   # kriging.py:345-357
    if len(kz) == 0:
        raise NoKnownNeighbors(f"no known voxel near {(x, y, z)}")
    coords = np.column_stack([kx + x0, ky + y0, kz + z0])
    (w,), _ = solve_systems([coords - np.array([x, y, z])], model, drift)
    pred = float(w @ data[coords[:, 2], coords[:, 1], coords[:, 0]].astype(np.float64))
    if clamp_range is None:
        known = data[~mask]
        clamp_range = (float(known.min()), float(known.max()))
    return float(np.clip(pred, clamp_range[0], clamp_range[1]))


def _fill_generic(grid, data_d, mask_d, model, drift, return_variance, on_dev, origin):
    """Non-plane masks on the device: ``vk_fill_generic`` (window schedule,
    distinct-pattern solves, per-voxel prediction; kriging.py:408-431)."""
    torch = _torch()
    lib = _lib.load()
    T, H, W = data_d.shape
    known = data_d[mask_d == 0]
    lo, hi = float(known.min().item()), float(known.max().item())   # kriging.py:475-479
    out_d = torch.empty_like(data_d)
    var_d = (torch.empty(data_d.shape, dtype=torch.float64, device=data_d.device)
             if return_variance else None)
    kind, m = _model_params(model)
    info = np.zeros(3, np.int64)
    raise_for_status(lib.vk_fill_generic(
        data_d.data_ptr(), mask_d.data_ptr(), T, H, W, _lib.KIND_IDS[kind],
        _lib.DRIFT_IDS[drift], m.ctypes.data, lo, hi, out_d.data_ptr(),
        var_d.data_ptr() if var_d is not None else None, info.ctypes.data,
        _stream_handle(None)))
    return _result(grid, out_d, var_d, on_dev, origin, return_variance)


def _result(grid, out_d, var_d, on_dev, origin, return_variance):
    """kriging.py:492-496: new grid, all-false mask, same origin_offset;
    numpy in -> numpy out, CUDA in -> CUDA out."""
    torch = _torch()
    if on_dev:
        out_grid = _like_grid(grid, out_d, torch.zeros(out_d.shape, dtype=torch.bool,
                                                       device=out_d.device), origin)
        return (out_grid, var_d) if return_variance else out_grid
    # host results land in page-locked memory from torch's caching host
    # allocator (no page faults on a fresh array, full PCIe rate; measured on
    # a C4 sub-part: 31.6 ms pageable vs 1.2 ms) and are returned as numpy
    # views of it
    def host(t):
        h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()
    out_grid = _like_grid(grid, host(out_d), np.zeros(tuple(out_d.shape), dtype=bool), origin)
    if return_variance:
        return out_grid, host(var_d)
    return out_grid


def fill_missing(grid: VolumeGrid, model: VariogramModel, drift="linear",
                 return_variance: bool = False, *, accum: str = "fp64"):
    """Fill every missing voxel by kriging from known voxels only.

    Known voxels pass through bit-exactly; predictions never read other
    predictions.  Host (numpy) grids come back as numpy, CUDA grids as CUDA
    tensors.  Plane-structured masks (the production case, kriging.py:485-487)
    take the streaming stencil kernels; any other mask takes the device
    per-voxel window path (kriging.py:488-490, 408-431).
    """
    torch = _torch()
    if callable(drift):
        raise DeviceUnsupported("a callable drift cannot cross the C ABI")
    kind, mparams = _model_params(model)
    data, mask, origin, on_dev = _grid_parts(grid)
    if on_dev:
        data_d, mask_d = data, mask.view(torch.uint8)
    else:
        data_d = _upload(data)
        mask_d = _upload(mask.view(np.uint8))
    T, H, W = data_d.shape
    counts = _scan_grid(data_d, mask_d)
    if counts[:, 2].any():
        raise ValueError("missing_mask out of sync with NaN sentinel")
    if counts[:, 3].any():
        raise ValueError("known voxels must be finite")
    n_missing = counts[:, 0].astype(np.int64)
    if n_missing.sum() == 0:                                 # kriging.py:469-473
        out = grid.copy() if hasattr(grid, "copy") else _like_grid(grid, data.clone() if on_dev
                                                                    else data.copy(), mask, origin)
        if return_variance:
            zeros = (torch.zeros(data_d.shape, dtype=torch.float64, device=data_d.device)
                     if on_dev else np.zeros(tuple(data.shape), dtype=np.float64))
            return out, zeros
        return out
    P = H * W
    if int((P - n_missing).sum()) == 0:                      # kriging.py:475-477
        raise NoKnownNeighbors("grid has no known voxels at all")
    known_z = np.nonzero(n_missing == 0)[0].astype(np.int32)
    if drift not in _lib.DRIFT_IDS:
        raise ValueError(f"unknown drift {drift!r}")
    if not np.all((n_missing == 0) | (n_missing == P)):
        # arbitrary mask: the per-voxel window path (kriging.py:488-490, 408-431)
        return _fill_generic(grid, data_d, mask_d, model, drift, return_variance, on_dev, origin)
    try:
        plan = cached_plan(height=H, width=W, depth=T, known_z=known_z.tolist(), n_subparts=1,
                           kind=kind, drift=drift, accum=accum, fit=False)
    except DeviceUnsupported:
        # a missing plane whose z window reaches more than NPMAX known planes:
        # the per-voxel path selects the same windows (in-plane 4, z extent
        # 4 -> 8 -> 16 until bracketed) with no plane limit
        return _fill_generic(grid, data_d, mask_d, model, drift, return_variance, on_dev, origin)
    lib = _lib.load()
    known_d = torch.empty((len(known_z), H, W), dtype=torch.float32, device=data_d.device)
    raise_for_status(lib.vk_gather_planes(data_d.data_ptr(), known_z.ctypes.data,
                                          len(known_z), P, known_d.data_ptr(),
                                          _stream_handle(None)))
    out_d = torch.empty((T, H, W), dtype=torch.float32, device=data_d.device)
    var_d = (torch.empty((T, H, W), dtype=torch.float64, device=data_d.device)
             if return_variance else None)
    plan.execute(known_d, out_d, var_d, models=mparams[None, :])
    plan.finish()
    return _result(grid, out_d, var_d, on_dev, origin, return_variance)
