"""Slice-stack input of the kriging path: the reference's manifest format and
``load_stack`` (io.py:26-143) with the sample decode and the stack
normalisation (``normalize_stack``, model.py:189-202) on the device.

* ``parse_manifest`` / ``write_manifest`` / ``StackManifest`` are host code
  with the reference's grammar, validation order and messages.
* Image files are decoded by Pillow on the host (entropy decoding stays on
  the CPU), in a thread pool, into their native integer
  samples: "L"/"P"/"1"/other -> ``convert("L")`` u8, "I;16" -> u16, "I" ->
  i32.  The raw samples (1-2 B per pixel instead of 4) are copied once to
  the device, where ``vk_normalize_stack`` converts them exactly as numpy
  does (f32(sample) / 255 or / 65535), reduces the global min/max and
  rescales to [0, 1] -- bit-identical to the reference's float32 stack.
  Mixed-mode stacks are decoded slice by slice (``vk_decode_samples``) and
  then normalised in place.
* Errors follow the reference's order: manifest errors, then per slice in
  manifest order ``ImageDecode`` / ``DimensionMismatch``, then the
  ``SliceStack`` checks.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import DimensionMismatch, ImageDecode, ManifestParse, raise_for_status
from .kriging import _stream_handle, _torch
from .model import AXIS_LABELS, SliceStack, check_stack_meta

SAMPLE_U8, SAMPLE_U16, SAMPLE_I32, SAMPLE_F32 = 0, 1, 2, 3     # VK_SAMPLE_*
_SAMPLE_DTYPE = {SAMPLE_U8: np.uint8, SAMPLE_U16: np.uint16, SAMPLE_I32: np.int32,
                 SAMPLE_F32: np.float32}


@dataclass
class StackManifest:
    """Parsed manifest (io.py:26-50): ordered slice paths, in-plane spacing,
    slice gap and axis label."""

    slice_files: list
    pixel_spacing_mm: tuple
    slice_gap_mm: float
    axis_label: str = "axial"

    def __post_init__(self):
        if not self.slice_files:
            raise ManifestParse("manifest lists no slices")
        if len(set(self.slice_files)) != len(self.slice_files):
            raise ManifestParse("duplicate slice paths in manifest")


def parse_manifest(path) -> StackManifest:
    """io.py:53-90: ``key = value`` lines, ``#`` comments, ordered ``slice``
    entries resolved against the manifest's directory."""
    path = Path(path)
    try:
        text = path.read_text(encoding="utf-8")
    except OSError as e:
        raise ManifestParse(f"cannot read manifest {path}: {e}") from e
    fields = {"pixel_spacing_mm": None, "slice_gap_mm": None, "axis": "axial"}
    files = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise ManifestParse(f"{path}:{lineno}: expected 'key = value'")
        key, value = key.strip(), value.strip()
        if key == "slice":
            files.append((path.parent / value).resolve())
        elif key == "pixel_spacing_mm":
            parts = value.split()
            if len(parts) != 2:
                raise ManifestParse(f"{path}:{lineno}: need two spacing values")
            fields[key] = (float(parts[0]), float(parts[1]))
        elif key == "slice_gap_mm":
            fields[key] = float(value)
        elif key == "axis":
            if value not in AXIS_LABELS:
                raise ManifestParse(f"{path}:{lineno}: unknown axis {value!r}")
            fields[key] = value
        else:
            raise ManifestParse(f"{path}:{lineno}: unknown key {key!r}")
    if fields["pixel_spacing_mm"] is None or fields["slice_gap_mm"] is None:
        raise ManifestParse(f"{path}: pixel_spacing_mm and slice_gap_mm are required")
    return StackManifest(files, fields["pixel_spacing_mm"], fields["slice_gap_mm"], fields["axis"])


def write_manifest(manifest: StackManifest, path) -> None:
    """io.py:93-105: slice paths relative to the manifest when possible."""
    path = Path(path)
    sx, sy = manifest.pixel_spacing_mm
    out = [f"pixel_spacing_mm = {sx} {sy}", f"slice_gap_mm = {manifest.slice_gap_mm}",
           f"axis = {manifest.axis_label}"]
    base = path.parent.resolve()
    for f in manifest.slice_files:
        try:
            rel = Path(f).relative_to(base)
        except ValueError:
            rel = Path(f)
        out.append(f"slice = {rel.as_posix()}")
    path.write_text("\n".join(out) + "\n", encoding="utf-8")


def decode_slice_samples(path):
    """The host half of ``_decode_slice`` (io.py:108-125): Pillow decode into
    the native integer samples -> (array [h, w], VK sample type)."""
    from PIL import Image, UnidentifiedImageError
    try:
        with Image.open(path) as img:
            img.load()
            if img.mode == "I;16":
                arr, kind = np.asarray(img, dtype=np.uint16), SAMPLE_U16
            elif img.mode == "I":
                arr, kind = np.asarray(img, dtype=np.int32), SAMPLE_I32
            else:                       # "L", "P", "1" and (defensively) colour
                arr, kind = np.asarray(img.convert("L"), dtype=np.uint8), SAMPLE_U8
    except (OSError, UnidentifiedImageError, ValueError) as e:
        raise ImageDecode(f"cannot decode {path}: {e}") from e
    if arr.ndim != 2:
        raise ImageDecode(f"{path}: expected a single-channel image")
    return arr, kind


def _n_samples(raw_dev, sample_type: int) -> int:
    """Samples in a device buffer of any torch dtype (raw bytes included)."""
    nbytes = raw_dev.numel() * raw_dev.element_size()
    size = np.dtype(_SAMPLE_DTYPE[int(sample_type)]).itemsize
    if nbytes % size:
        raise ValueError(f"{nbytes} bytes is not a whole number of {size}-byte samples")
    return nbytes // size


def decode_samples(samples_dev, sample_type: int):
    """Device f32 decode of raw samples (``vk_decode_samples``) -> flat f32."""
    torch = _torch()
    n = _n_samples(samples_dev, sample_type)
    out = torch.empty(n, dtype=torch.float32, device=samples_dev.device)
    raise_for_status(_lib.load().vk_decode_samples(samples_dev.data_ptr(), int(sample_type), n,
                                                   out.data_ptr(), _stream_handle(None)))
    return out


def _normalize_dev(raw_dev, sample_type: int, out=None):
    """vk_normalize_stack over a contiguous device buffer -> flat f32 (or `out`)."""
    torch = _torch()
    n = _n_samples(raw_dev, sample_type)
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=raw_dev.device)
    raise_for_status(_lib.load().vk_normalize_stack(raw_dev.data_ptr(), int(sample_type), n,
                                                    out.data_ptr(), None, _stream_handle(None)))
    return out


def normalize_stack(raw: SliceStack) -> SliceStack:
    """model.py:189-202 on the device: global min -> 0, max -> 1 in float32;
    a constant stack maps to zeros.  Host stacks are uploaded first."""
    torch = _torch()
    src = raw.slices if raw.on_device else torch.from_numpy(raw.slices).cuda()
    return SliceStack(_normalize_dev(src, SAMPLE_F32).view(src.shape), raw.pixel_spacing, raw.slice_gap_mm, raw.axis_label)


def _decode_all(files, workers):
    """Pillow decodes in a thread pool; results and errors surface in
    manifest order, so the first failing slice is the reference's."""
    workers = workers or min(32, os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=max(1, workers)) as ex:
        futs = [ex.submit(decode_slice_samples, f) for f in files]
        out, shape = [], None
        for f, fut in zip(files, futs):
            arr, kind = fut.result()
            if shape is None:
                shape = arr.shape
            elif arr.shape != shape:
                for g in futs:
                    g.cancel()
                raise DimensionMismatch(f"{f}: slice is {arr.shape}, expected {shape}")
            out.append((arr, kind))
    return out, shape


def load_stack(manifest_path, device: bool = False, workers: int | None = None) -> SliceStack:
    """io.py:128-143: parse, decode, stack and normalise (on the device).  The
    result's ``slices`` is a numpy float32 [n, h, w] array like the
    reference's; ``device=True`` keeps it as the CUDA tensor the kriging path
    consumes."""
    manifest = parse_manifest(manifest_path)
    decoded, (h, w) = _decode_all(manifest.slice_files, workers)
    n = len(decoded)
    check_stack_meta((n, h, w), manifest.pixel_spacing_mm, manifest.slice_gap_mm, manifest.axis_label)
    torch = _torch()
    kinds = {k for _, k in decoded}
    if len(kinds) == 1:
        kind = kinds.pop()
        dt = _SAMPLE_DTYPE[kind]
        host = torch.empty(n * h * w * np.dtype(dt).itemsize, dtype=torch.uint8, pin_memory=True)
        view = host.numpy().view(dt).reshape(n, h, w)
        for i, (arr, _) in enumerate(decoded):
            view[i] = arr
        raw = host.cuda(non_blocking=True)
        data = _normalize_dev(raw, kind).view(n, h, w)
    else:
        data = torch.empty((n, h, w), dtype=torch.float32, device="cuda")
        for i, (arr, kind) in enumerate(decoded):
            raw_i = torch.from_numpy(np.array(arr).view(np.uint8)).cuda()
            raise_for_status(_lib.load().vk_decode_samples(raw_i.data_ptr(), kind, h * w, data[i].data_ptr(),
                                                           _stream_handle(None)))
        _normalize_dev(data, SAMPLE_F32, out=data)
    stack = SliceStack(data, manifest.pixel_spacing_mm, manifest.slice_gap_mm, manifest.axis_label)
    if not device:
        stack = SliceStack(stack.slices.cpu().numpy(), stack.pixel_spacing, stack.slice_gap_mm, stack.axis_label)
    return stack
