"""The reference's binary volume format (io.py:146-200) with the heavy work on
the device: ``VOLKRIG\\0`` magic, ``<I3I3i`` header (version, dx, dy, dz,
origin), the f32 payload in [z, y, x] C order, ``np.packbits`` of the missing
mask, and a trailing CRC-32 of everything before it.

* ``save_volume`` produces the same bytes as the reference: the mask is
  packed by ``vk_packbits`` and the CRC runs over the device-resident payload
  and packed mask with ``vk_crc32`` (continuing the header's CRC exactly as
  ``zlib.crc32`` would), so an 8.6 GB output volume never needs a host pass
  besides the final write.  The file is written to ``path + ".tmp"`` and
  renamed into place (io.py:160-167).
* ``load_volume`` checks size, magic, version and length on the host in the
  reference's order (io.py:170-186, ``CorruptHeader``), uploads the body once
  and verifies the CRC on the device (``ChecksumMismatch``), then unpacks the
  mask there.  The default returns numpy arrays like the reference;
  ``device=True`` keeps the grid on the GPU.
"""

from __future__ import annotations

import ctypes as C
import struct
import zlib
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ChecksumMismatch, CorruptHeader, InvalidGrid, Io, raise_for_status
from .kriging import _stream_handle, _torch
from .model import VolumeGrid

VOLUME_MAGIC = b"VOLKRIG\x00"        # io.py:22
VOLUME_VERSION = 1                   # io.py:23
_HEAD = "<I3I3i"
HEAD_LEN = len(VOLUME_MAGIC) + struct.calcsize(_HEAD)


def crc32(data_dev, n_bytes: int, crc_in: int = 0) -> int:
    """zlib.crc32(bytes of a device buffer, crc_in) computed on the GPU."""
    out = C.c_uint32()
    raise_for_status(_lib.load().vk_crc32(data_dev.data_ptr() if n_bytes else None, int(n_bytes),
                                          int(crc_in) & 0xFFFFFFFF, C.byref(out),
                                          _stream_handle(None)))
    return int(out.value)


def packbits(mask_dev):
    """np.packbits(mask.reshape(-1)) on the device (uint8 tensor)."""
    torch = _torch()
    n = mask_dev.numel()
    bits = torch.empty((n + 7) // 8, dtype=torch.uint8, device=mask_dev.device)
    raise_for_status(_lib.load().vk_packbits(mask_dev.contiguous().view(torch.uint8).data_ptr(), n,
                                             bits.data_ptr(), _stream_handle(None)))
    return bits


def unpackbits(bits_dev, n: int):
    torch = _torch()
    mask = torch.empty(n, dtype=torch.uint8, device=bits_dev.device)
    raise_for_status(_lib.load().vk_unpackbits(bits_dev.data_ptr(), n, mask.data_ptr(),
                                               _stream_handle(None)))
    return mask.view(torch.bool)


def save_volume(grid: VolumeGrid, path) -> None:
    """io.py:146-167."""
    torch = _torch()
    if grid.n_voxels == 0:
        raise InvalidGrid("refusing to save a volume with empty dims")
    grid.validate()
    dx, dy, dz = grid.dims
    header = VOLUME_MAGIC + struct.pack(_HEAD, VOLUME_VERSION, dx, dy, dz, *grid.origin_offset)
    if grid.on_device:
        data_d, mask_d = grid.data, grid.missing_mask
    else:
        data_d = torch.from_numpy(grid.data).cuda()
        mask_d = torch.from_numpy(grid.missing_mask).cuda()
    n = grid.n_voxels
    bits_d = packbits(mask_d)
    crc = zlib.crc32(header)                      # 36 header bytes on the host
    crc = crc32(data_d, 4 * n, crc)
    crc = crc32(bits_d, bits_d.numel(), crc)
    payload = data_d.cpu().numpy() if grid.on_device else grid.data
    try:
        tmp = Path(str(path) + ".tmp")
        with open(tmp, "wb") as fh:
            fh.write(header)
            fh.write(np.ascontiguousarray(payload, dtype="<f4").tobytes())
            fh.write(bits_d.cpu().numpy().tobytes())
            fh.write(struct.pack("<I", crc))
        tmp.replace(path)
    except OSError as e:
        raise Io(f"cannot write volume {path}: {e}") from e


def parse_header(blob: bytes, path="<bytes>"):
    """Host checks of io.py:175-186; returns (dims (dx, dy, dz), origin)."""
    if len(blob) < HEAD_LEN + 4:
        raise CorruptHeader(f"{path}: truncated volume file")
    if blob[:len(VOLUME_MAGIC)] != VOLUME_MAGIC:
        raise CorruptHeader(f"{path}: bad magic bytes")
    version, dx, dy, dz, ox, oy, oz = struct.unpack_from(_HEAD, blob, len(VOLUME_MAGIC))
    if version != VOLUME_VERSION:
        raise CorruptHeader(f"{path}: unsupported volume version {version}")
    n = dx * dy * dz
    expected = HEAD_LEN + 4 * n + (n + 7) // 8 + 4
    if len(blob) != expected:
        raise CorruptHeader(f"{path}: size {len(blob)} != expected {expected} for dims {(dx, dy, dz)}")
    return (dx, dy, dz), (ox, oy, oz)


def load_volume(path, device: bool = False) -> VolumeGrid:
    """io.py:170-200; the CRC check and mask unpacking run on the GPU."""
    try:
        blob = Path(path).read_bytes()
    except OSError as e:
        raise Io(f"cannot read volume {path}: {e}") from e
    (dx, dy, dz), origin = parse_header(blob, path)
    torch = _torch()
    n = dx * dy * dz
    body = np.frombuffer(blob, dtype=np.uint8, offset=HEAD_LEN, count=len(blob) - HEAD_LEN - 4)
    body_d = torch.from_numpy(body.copy()).cuda()
    crc = crc32(body_d, body_d.numel(), zlib.crc32(blob[:HEAD_LEN]))
    if crc != struct.unpack_from("<I", blob, len(blob) - 4)[0]:
        raise ChecksumMismatch(f"{path}: CRC mismatch")
    data_d = body_d[:4 * n].view(torch.float32).reshape(dz, dy, dx)
    mask_d = unpackbits(body_d[4 * n:], n).reshape(dz, dy, dx)
    if device:
        return VolumeGrid(data_d, mask_d, origin)
    return VolumeGrid(data_d.cpu().numpy(), mask_d.cpu().numpy(), origin)
