"""Z sub-part sharding across the GPUs of one node (one process per GPU).

Sub-parts are independent once each holds its trailing one-known-slice halo
(SURVEY.md 8e), so a rank owns a contiguous run of parts and the only data
exchange is that halo: rank r needs the first known slice of rank r+1.  It is
sent with one ``torch.distributed`` send/recv pair (NCCL over NVLink on GPUs,
gloo in the CPU tests).  The reconstructed volume stays sharded; ``gather``
collects the core planes on rank 0 when a caller wants the whole volume (the
gather is reported separately from the kriging path).

Two partitions are provided:

* ``strong_shard``: a given stack of K slices and S parts split over G ranks
  (rank r owns parts [r*S/G, (r+1)*S/G)), bit-identical to the single-device
  result because every part sees exactly the same data, pairs and model;
* weak scaling (bench.py): every rank owns its own K_local slices; the
  global volume is their concatenation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    k0: int            # first owned known slice (global index)
    k1: int            # last owned known slice (inclusive, without halo)
    has_halo: bool     # receives slice k1 + 1 from rank + 1
    part0: int         # first owned sub-part
    n_parts: int
    part_len: int      # q (global), so local parts match the global ones

    @property
    def n_local(self) -> int:
        """Known slices in the local stack, halo included."""
        return self.k1 - self.k0 + 1 + int(self.has_halo)


def strong_shard(n_known: int, n_parts: int, rank: int, world: int) -> Shard:
    if n_parts % world:
        raise ValueError("n_subparts must be divisible by the number of ranks")
    q = n_known // n_parts
    per = n_parts // world
    p0 = rank * per
    k0 = p0 * q
    last = rank == world - 1
    k1 = n_known - 1 if last else (p0 + per) * q - 1
    return Shard(rank, world, k0, k1, not last, p0, per, q)


def exchange_halo(first_plane, rank: int, world: int, group=None, out=None):
    """Send our first known plane to rank-1; receive rank+1's (or None) into
    ``out`` when given (e.g. the stack's trailing halo slot, no extra copy)."""
    import torch
    import torch.distributed as dist
    ops = []
    halo = None
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, first_plane.contiguous(), rank - 1, group))
    if rank < world - 1:
        halo = out if out is not None else torch.empty_like(first_plane)
        ops.append(dist.P2POp(dist.irecv, halo, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return halo


def local_stack(owned, halo):
    """Owned slices [n, H, W] plus the halo slice appended (if any)."""
    import torch
    return owned if halo is None else torch.cat([owned, halo[None]], dim=0)


def core_planes(volume, factor: int, has_halo: bool):
    """Drop the trailing halo plane (a known plane owned by the next rank)."""
    return volume[:-1] if has_halo else volume


def gather_volume(core, rank: int, world: int, group=None):
    """Concatenate every rank's core planes on rank 0 (others get None)."""
    import torch
    import torch.distributed as dist
    shapes = [None] * world
    dist.all_gather_object(shapes, tuple(core.shape), group=group)
    if rank == 0:
        parts = [core]
        for src in range(1, world):
            buf = torch.empty(shapes[src], dtype=core.dtype, device=core.device)
            dist.recv(buf, src=src, group=group)
            parts.append(buf)
        return torch.cat(parts, dim=0)
    dist.send(core.contiguous(), dst=0, group=group)
    return None


class NativeComm:
    """The C ABI's NCCL communicator (``vk_comm_*``): the halo exchange and
    the gather of core planes as grouped send / receive on a CUDA stream,
    without torch.distributed on the data path.  Rank 0 creates the unique
    id; with more than one rank it is broadcast over ``group``
    (torch.distributed, any backend)."""

    def __init__(self, rank: int, world: int, group=None):
        import ctypes as C
        from . import _lib
        from .errors import raise_for_status
        self._lib, self._raise = _lib.load(), raise_for_status
        self.rank, self.world = int(rank), int(world)
        idb = (C.c_ubyte * 128)()
        if self.rank == 0:
            self._raise(self._lib.vk_comm_unique_id(idb))
        if self.world > 1:
            import torch.distributed as dist
            box = [bytes(idb)]
            dist.broadcast_object_list(box, src=0, group=group)
            C.memmove(idb, box[0], 128)
        h = C.c_void_p()
        self._raise(self._lib.vk_comm_create(idb, self.world, self.rank, C.byref(h)))
        self._h = h

    def _stream(self, stream):
        import torch
        return (stream or torch.cuda.current_stream()).cuda_stream

    def halo(self, first_plane, out=None, stream=None):
        """Send ``first_plane`` to rank - 1; receive rank + 1's into ``out``
        (allocated when None) on ranks below the last; returns it or None."""
        import torch
        first_plane = first_plane.contiguous()
        if self.rank < self.world - 1 and out is None:
            out = torch.empty_like(first_plane)
        self._raise(self._lib.vk_halo_exchange(
            self._h, first_plane.data_ptr(), out.data_ptr() if out is not None else None,
            first_plane.numel(), self._stream(stream)))
        return out if self.rank < self.world - 1 else None

    def gather(self, core, counts, stream=None):
        """Rank 0: every rank's ``core`` (counts[r] floats) concatenated in
        rank order; other ranks send theirs and get None."""
        import ctypes as C
        import torch
        core = core.contiguous()
        cnt = (C.c_int64 * self.world)(*[int(c) for c in counts])
        out = torch.empty(int(sum(counts)), dtype=torch.float32, device=core.device) \
            if self.rank == 0 else None
        self._raise(self._lib.vk_gather_core(self._h, core.data_ptr(), cnt,
                                             out.data_ptr() if out is not None else None,
                                             self._stream(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vk_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def reconstruct_sharded(owned, factor: int, shard: Shard, reconstruct=None, group=None,
                        gather: bool = True, **kw):
    """Halo exchange -> local Z-part kriging -> (optional) gather on rank 0.

    ``reconstruct(local_stack, factor, n_parts, part_len) -> volume`` defaults
    to the device path (``ZPartKriging``); tests inject the CPU oracle to
    check the host-side partition/exchange/merge logic with gloo.
    """
    halo = exchange_halo(owned[0], shard.rank, shard.world, group)
    stack = local_stack(owned, halo)
    if reconstruct is None:
        reconstruct = _device_reconstruct
    vol = reconstruct(stack, factor, shard.n_parts, shard.part_len, **kw)
    core = core_planes(vol, factor, shard.has_halo)
    if not gather:
        return core
    return gather_volume(core, shard.rank, shard.world, group)


def _device_reconstruct(stack, factor, n_parts, part_len, **kw):
    from .block_pipeline import ZPartKriging
    K, H, W = stack.shape
    zk = ZPartKriging(K, H, W, factor, n_parts, part_len=part_len, **kw)
    out, _ = zk.run(stack.contiguous())
    zk.finish()
    return out


def global_part_ranges(n_known: int, n_parts: int) -> list[tuple[int, int]]:
    q = n_known // n_parts
    return [(s * q, (s + 1) * q if s < n_parts - 1 else n_known - 1) for s in range(n_parts)]


def check_cover(shards: list[Shard], n_known: int) -> None:
    """Owned ranges tile [0, K) exactly (merge invariant)."""
    cover = np.zeros(n_known, np.int32)
    for s in shards:
        cover[s.k0:s.k1 + 1] += 1
    if not np.all(cover == 1):
        raise AssertionError("shards do not tile the stack")
